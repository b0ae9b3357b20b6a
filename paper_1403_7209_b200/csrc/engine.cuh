// Loop engine: one templated CUDA kernel family per loop *shape*, specialised
// at compile time for each hand-written functor (the B200 counterpart of the
// per-loop code OP2 generates; reference execution semantics executor.py:
// 149-275, plan consumption plan.py:30-45).
//
// A functor declares its argument signature (kind, access mode, dim, type)
// and a device `apply(consts, view0, view1, ...)`.  Views are
//   * Ref<T>/Ref<const T>  — strided references straight into HBM for
//     direct args, indirect READ args and (phased mode) indirect WRITE/RW
//     args; loads are issued at first use, so the compiler schedules them
//     and register pressure stays bounded for wide dats;
//   * T*                   — a register array: increments of an indirect INC
//     argument (applied colour by colour after the element is computed) and
//     global INC/MIN/MAX accumulators (block-reduced afterwards).
//
// Kernels
//   k_direct  — loops without indirect writes: one launch over all plan
//               blocks, per-block reduction partials.
//   k_staged  — loops whose only indirect writes are INC and bs <= blockDim:
//               every thread computes its element at once, then element
//               colour phases (separated by __syncthreads) apply the
//               register increments with plain read-modify-write.  One
//               launch per block colour; blocks of one colour share no
//               target, so no atomics are needed and the result is
//               deterministic run to run.
//   k_phased  — general case (indirect WRITE/RW, or bs > blockDim): each
//               element executes entirely inside its colour phase.
// Global reductions: warp shuffle -> shared -> one partial per plan block;
// k_combine folds the partials in a fixed order onto the initial value.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cuda/std/limits>
#include <cuda/std/tuple>
#include <cuda/std/type_traits>
#include <cuda/std/utility>

namespace ml {

enum : int { KD = 0, KI = 1, KG = 2 };                        // direct / indirect / global
enum : int { MR = 0, MW = 1, MRW = 2, MINC = 3, MMIN = 4, MMAX = 5 };
constexpr int MAX_ARGS = 16;

// Programmatic dependent launch: the hot kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization, so a kernel's CTAs can
// be resident while its predecessor on the stream drains; each such kernel
// waits (griddepcontrol.wait) for the predecessor's completion — and memory —
// before touching any data.  Without the attribute the wait is a no-op.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
bool pdl_enabled();
bool pass2_warp();

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
};

struct Consts {
    double f[4];
    int64_t i[4];
};

constexpr int MAX_GROUPS = 2;

// Shared-memory staging of indirect increments (OP2-style): per block, the
// sorted unique targets of each INC dat ("group") and, per element and INC
// argument, the target's position in that list.
struct Staging {
    int32_t group[MAX_ARGS];             // staging group of each arg (-1: none)
    int32_t leader[MAX_ARGS];            // 1 on the arg that writes its group back
    const int32_t *off[MAX_GROUPS];      // [nblocks+1] offsets into list
    const int32_t *list[MAX_GROUPS];     // unique targets, ascending per block
    const uint16_t *loc[MAX_ARGS];       // [n] local position of the arg's target
    int32_t umax[MAX_GROUPS];            // max unique targets per block (smem stride)
    int32_t soff[MAX_GROUPS];            // byte offset of the group in dynamic smem
    // segmented mode: private slot per (element, INC arg); per unique target the
    // contributing slots in element order (src = arg position * 256 + element)
    const int32_t *toff[MAX_GROUPS];     // [total+1] into src (global target index)
    const uint16_t *src[MAX_GROUPS];
    int32_t gpos[MAX_ARGS];              // position of the arg inside its group
    // arrival mode: shared targets go through per-block partial slots; the last
    // block to arrive (atomic counter) folds them in block order
    const int32_t *pslot[MAX_GROUPS];    // [total] partial slot per list entry (-1: sole block)
    const int32_t *poff[MAX_GROUPS];     // [targets] first slot of a shared target
    const int32_t *nblk[MAX_GROUPS];     // [targets] blocks touching the target
    int32_t *count[MAX_GROUPS];          // [targets] arrivals (back to 0 after each run)
    void *partial[MAX_GROUPS];           // [slots][dim]
    int32_t foff[MAX_GROUPS];            // byte offset of the finaliser list in dynamic smem
};

// Tile schedule (csrc/host_tile.cpp): per tile, the staged target list (owned
// first), the elements it evaluates with their local target indices per map
// column, element colours (bit 7: reduction owner) and the colour count.
constexpr int MAX_TGROUPS = 8;
struct TileParams {
    const int32_t *list_off, *nown, *list, *elem_off, *elem, *ncol;
    const uint16_t *loc;
    const uint8_t *ecol;
    int32_t arity;
    int32_t nread, ninc;                 // staged READ dats, accumulated INC dats
    int32_t garg[MAX_TGROUPS];           // an argument of each group (read groups, then INC)
    int32_t gdim[MAX_TGROUPS];           // components of each group's dat
    int8_t grp[MAX_ARGS];                // group of each indirect argument
    int8_t slot[MAX_ARGS];               // map column of each indirect argument
    // tile-gather variant: per owned target, (element-in-tile, column) incidences
    const int32_t *inc_base, *inc_off;
    const uint16_t *inc_k;
    const uint8_t *inc_c;
    int32_t red_col;                     // column whose incidence counts the element in reductions
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
    // own-row staging: READ dats read through the first INC argument's column
    // (the target itself) are copied once per target to shared memory
    int32_t own_ngrp;
    int32_t own_garg[MAX_TGROUPS], own_gdim[MAX_TGROUPS], own_goff[MAX_TGROUPS];
    int8_t own_grp[MAX_ARGS];
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
    Staging st;
    int64_t n;
    int64_t rlim;               // elements >= rlim do not contribute to reductions
    int32_t bs;
    const int32_t *blocks;      // block ids of this launch (nullptr: identity)
    const int32_t *dep_off;     // dataflow: per block, lower-colour conflicting blocks
    const int32_t *dep_list;
    int32_t *flags;             // dataflow: [nblocks] done flags + queue counter at [nblocks]
    int32_t nqueue;             // dataflow: number of blocks in the queue
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
    // fold schedule: per (element, INC-arg position) increment slots, element-major
    void *g_buf;
    int32_t g_nw;               // INC arguments per element
    TileParams t;
    PFoldParams pf;
};

// strided view of one element's components
template <class T>
struct Ref {
    T *p;
    int64_t sc;
    __device__ __forceinline__ T &operator[](int c) const { return p[c * sc]; }
};

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

// ---- per-argument slot --------------------------------------------------------
// MODE 0: no staging (views into HBM); 1: indirect INC staged in registers and
// applied to HBM in colour phases; 2: staged in registers, applied to shared
// memory in colour phases, written back once per block.
// MODE 3 (ST_SEG): the functor increments a private shared-memory slot of its
// own (no registers held, no phases); the write-back sums each target's slots
// in element order — a deterministic segmented reduction.
// MODE 4 (ST_GATHER): target-centric schedule — INC and WRITE indirect args
// are staged in registers (zero-initialised); the kernel keeps one of them.
// MODE 5 (ST_TILE): tile schedule — indirect READ args view the tile's staged
// copy in shared memory, INC args are staged in registers and added in colour
// phases to the tile's shared-memory accumulators of owned targets (increments
// of targets owned by another tile are dropped: that tile evaluates the
// element too).
enum : int { ST_NONE = 0, ST_REG = 1, ST_SMEM = 2, ST_SEG = 3, ST_GATHER = 4, ST_TILE = 5 };

template <class A, int MODE>
struct Slot {
    using T = typename A::type;
    static constexpr bool is_global = A::kind == KG;
    static constexpr bool is_reduce = is_global && A::mode != MR;
    static constexpr bool is_inc = A::kind == KI && A::mode == MINC;
    static constexpr bool seg = is_inc && MODE == ST_SEG;
    static constexpr bool is_ind_write = A::kind == KI && A::mode == MW;
    static constexpr bool staged = (is_inc && MODE != ST_NONE && MODE != ST_SEG) || is_reduce ||
                                   (is_ind_write && MODE == ST_GATHER);

    T acc[staged ? A::dim : 1];
    T bak[is_reduce ? A::dim : 1];
    T *ptr;          // element base pointer (HBM or shared memory)
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
    __device__ __forceinline__ void init_elem(const LaunchParams &p, int i, int64_t e, char *smem) {
        if constexpr (!is_global) {
            if constexpr (is_inc && MODE == ST_SMEM) {
                const int g = p.st.group[i];
                ptr = reinterpret_cast<T *>(smem + p.st.soff[g]) + __ldg(p.st.loc[i] + e);
                sc = p.st.umax[g];
            } else if constexpr (seg) {
                const int g = p.st.group[i];
                ptr = reinterpret_cast<T *>(smem + p.st.soff[g]) +
                      int64_t(p.st.gpos[i]) * A::dim * blockDim.x + threadIdx.x;
                sc = blockDim.x;
#pragma unroll
                for (int c = 0; c < A::dim; ++c) ptr[c * sc] = T(0);
            } else {
                const ArgRt &r = p.a[i];
                const int64_t t = A::kind == KI ? int64_t(__ldg(r.map + e)) : e;
                ptr = static_cast<T *>(r.data) + t * r.se;
                sc = r.sc;
            }
            if constexpr (staged) {
#pragma unroll
                for (int c = 0; c < A::dim; ++c) acc[c] = T(0);
            }
        }
    }
    // pass-1 element record (PFoldParams::rec): indirect targets from the record
    __device__ __forceinline__ void init_elem_rec(const LaunchParams &p, int i, int64_t e, const int32_t *rk) {
        if constexpr (!is_global) {
            const ArgRt &r = p.a[i];
            const int64_t t = A::kind == KI ? int64_t(__ldg(rk + p.pf.rcol[i])) : e;
            ptr = static_cast<T *>(r.data) + t * r.se;
            sc = r.sc;
            if constexpr (staged) {
#pragma unroll
                for (int c = 0; c < A::dim; ++c) acc[c] = T(0);
            }
        }
    }
    // gather schedule with CTA-local staging: READ args whose target lies in
    // the CTA's range [t0, t0 + blockDim) read the staged copy
    // tile schedule: `gb` are the group bases in shared memory, U the staged
    // count (component stride of READ copies), C the owned count
    __device__ __forceinline__ void init_tile(const LaunchParams &p, int i, int64_t e, const uint16_t *locs,
                                              char *const *gb, int U, int C) {
        if constexpr (!is_global) {
            if constexpr (A::kind == KI) {
                const int l = locs[p.t.slot[i]];
                T *base = reinterpret_cast<T *>(gb[p.t.grp[i]]);
                if constexpr (is_inc) {
                    ptr = l < C ? base + l : nullptr;
                    sc = C;
                } else {
                    ptr = base + l;
                    sc = U;
                }
            } else {
                const ArgRt &r = p.a[i];
                ptr = static_cast<T *>(r.data) + e * r.se;
                sc = r.sc;
            }
            if constexpr (staged) {
#pragma unroll
                for (int c = 0; c < A::dim; ++c) acc[c] = T(0);
            }
        }
    }
    __device__ __forceinline__ auto view() {
        if constexpr (staged) {
            return static_cast<T *>(acc);
        } else if constexpr (A::mode == MR) {
            return Ref<const T>{ptr, sc};
        } else {
            return Ref<T>{ptr, sc};
        }
    }
    __device__ __forceinline__ void apply_staged() {
        if constexpr (staged && !is_global) {
            if constexpr (MODE == ST_TILE)
                if (!ptr) return;
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
    // shared memory -> HBM, once per block (MODE 2, group leader only)
    __device__ __forceinline__ void zero_smem(const LaunchParams &p, int i, int32_t b, char *smem) {
        if constexpr (is_inc && MODE == ST_SMEM) {
            const int g = p.st.group[i];
            if (!p.st.leader[i]) return;
            const int32_t lo = p.st.off[g][b], u = p.st.off[g][b + 1] - lo, um = p.st.umax[g];
            T *s = reinterpret_cast<T *>(smem + p.st.soff[g]);
            for (int k = threadIdx.x; k < u * A::dim; k += blockDim.x) s[(k / u) * um + (k % u)] = T(0);
        }
    }
    __device__ __forceinline__ void write_back(const LaunchParams &p, int i, int32_t b, char *smem) {
        if constexpr (is_inc && MODE == ST_SMEM) {
            const int g = p.st.group[i];
            if (!p.st.leader[i]) return;
            const int32_t lo = p.st.off[g][b], u = p.st.off[g][b + 1] - lo, um = p.st.umax[g];
            const T *s = reinterpret_cast<const T *>(smem + p.st.soff[g]);
            const int32_t *__restrict__ list = p.st.list[g] + lo;
            const ArgRt &r = p.a[i];
            T *d = static_cast<T *>(r.data);
            const int total = u * A::dim;
            const bool aos = r.sc == 1 && A::dim > 1;   // AOS: component-fastest is contiguous
            constexpr int U = 4;
            for (int k0 = threadIdx.x; k0 < total; k0 += U * blockDim.x) {
                int64_t addr[U];
                T val[U];
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const int k = k0 + q * blockDim.x;
                    if (k < total) {
                        const int c = aos ? k % A::dim : k / u, j = aos ? k / A::dim : k % u;
                        addr[q] = int64_t(__ldg(list + j)) * r.se + c * r.sc;
                        val[q] = s[c * um + j];
                    }
                }
#pragma unroll
                for (int q = 0; q < U; ++q)
                    if (k0 + q * blockDim.x < total) val[q] += __ldcg(d + addr[q]);
#pragma unroll
                for (int q = 0; q < U; ++q)
                    if (k0 + q * blockDim.x < total) d[addr[q]] = val[q];
            }
        } else if constexpr (seg) {
            const int g = p.st.group[i];
            if (!p.st.leader[i]) return;
            const int32_t lo = p.st.off[g][b], u = p.st.off[g][b + 1] - lo;
            const T *s = reinterpret_cast<const T *>(smem + p.st.soff[g]);
            const int32_t *__restrict__ list = p.st.list[g] + lo;
            const int32_t *__restrict__ toff = p.st.toff[g] + lo;
            const uint16_t *__restrict__ src = p.st.src[g];
            const ArgRt &r = p.a[i];
            T *d = static_cast<T *>(r.data);
            const int total = u * A::dim, nt = blockDim.x;
            const bool aos = r.sc == 1 && A::dim > 1;
            constexpr int U = 4;
            for (int k0 = threadIdx.x; k0 < total; k0 += U * nt) {
                int64_t addr[U];
                T val[U];
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const int k = k0 + q * nt;
                    if (k < total) {
                        const int c = aos ? k % A::dim : k / u, j = aos ? k / A::dim : k % u;
                        addr[q] = int64_t(__ldg(list + j)) * r.se + c * r.sc;
                        T acc = T(0);
                        for (int m = __ldg(toff + j), me = __ldg(toff + j + 1); m < me; ++m) {
                            const int v = __ldg(src + m);
                            acc += s[((v >> 8) * A::dim + c) * nt + (v & 255)];
                        }
                        val[q] = acc;
                    }
                }
#pragma unroll
                for (int q = 0; q < U; ++q)
                    if (k0 + q * nt < total) val[q] = __ldcg(d + addr[q]) + val[q];
#pragma unroll
                for (int q = 0; q < U; ++q)
                    if (k0 + q * nt < total) d[addr[q]] = val[q];
            }
        }
    }

    // ---- arrival mode (segmented slots, no block colours) ------------------------
    // phase 1: per (target, component) fold this block's slots in element order;
    // a target owned by this block alone is updated in HBM, a shared one writes
    // its block sum into the target's partial slot for this block.
    __device__ __forceinline__ void arrive_sums(const LaunchParams &p, int i, int32_t b, char *smem) {
        if constexpr (seg) {
            const int g = p.st.group[i];
            if (!p.st.leader[i]) return;
            const int32_t lo = p.st.off[g][b], u = p.st.off[g][b + 1] - lo;
            const T *s = reinterpret_cast<const T *>(smem + p.st.soff[g]);
            const int32_t *__restrict__ list = p.st.list[g] + lo;
            const int32_t *__restrict__ toff = p.st.toff[g] + lo;
            const int32_t *__restrict__ pslot = p.st.pslot[g] + lo;
            const uint16_t *__restrict__ src = p.st.src[g];
            T *part = static_cast<T *>(p.st.partial[g]);
            const ArgRt &r = p.a[i];
            T *d = static_cast<T *>(r.data);
            const int total = u * A::dim, nt = blockDim.x;
            const bool aos = r.sc == 1 && A::dim > 1;
            for (int k = threadIdx.x; k < total; k += nt) {
                const int c = aos ? k % A::dim : k / u, j = aos ? k / A::dim : k % u;
                T acc = T(0);
                for (int m = __ldg(toff + j), me = __ldg(toff + j + 1); m < me; ++m) {
                    const int v = __ldg(src + m);
                    acc += s[((v >> 8) * A::dim + c) * nt + (v & 255)];
                }
                const int32_t ps = __ldg(pslot + j);
                if (ps < 0) {
                    const int64_t a = int64_t(__ldg(list + j)) * r.se + c * r.sc;
                    d[a] = __ldcg(d + a) + acc;
                } else {
                    __stcg(part + int64_t(ps) * A::dim + c, acc);
                }
            }
        }
    }
    // phase 2 (after a fence + barrier): count this block's arrival at every
    // shared target; the last arriver queues the target for finalisation and
    // resets its counter for the next run.
    __device__ __forceinline__ void arrive_count(const LaunchParams &p, int i, int32_t b, char *smem,
                                                 int *nfin) {
        if constexpr (seg) {
            const int g = p.st.group[i];
            if (!p.st.leader[i]) return;
            const int32_t lo = p.st.off[g][b], u = p.st.off[g][b + 1] - lo;
            int32_t *fin = reinterpret_cast<int32_t *>(smem + p.st.foff[g]);
            for (int j = threadIdx.x; j < u; j += blockDim.x) {
                if (__ldg(p.st.pslot[g] + lo + j) < 0) continue;
                const int32_t t = __ldg(p.st.list[g] + lo + j);
                const int32_t need = __ldg(p.st.nblk[g] + t);
                if (atomicAdd(p.st.count[g] + t, 1) == need - 1) {
                    p.st.count[g][t] = 0;
                    fin[atomicAdd(nfin + g, 1)] = t;
                }
            }
        }
    }
    // phase 3: fold the partial slots of finalised targets in block order
    __device__ __forceinline__ void arrive_final(const LaunchParams &p, int i, char *smem, const int *nfin) {
        if constexpr (seg) {
            const int g = p.st.group[i];
            if (!p.st.leader[i]) return;
            const int nf = nfin[g];
            const int32_t *fin = reinterpret_cast<const int32_t *>(smem + p.st.foff[g]);
            const T *part = static_cast<const T *>(p.st.partial[g]);
            const ArgRt &r = p.a[i];
            T *d = static_cast<T *>(r.data);
            for (int k = threadIdx.x; k < nf * A::dim; k += blockDim.x) {
                const int c = k % A::dim;
                const int32_t t = fin[k / A::dim];
                const int32_t o = __ldg(p.st.poff[g] + t), nb = __ldg(p.st.nblk[g] + t);
                T acc = T(0);
                for (int q = 0; q < nb; ++q) acc += __ldcg(part + int64_t(o + q) * A::dim + c);
                const int64_t a = int64_t(t) * r.se + c * r.sc;
                d[a] = __ldcg(d + a) + acc;
            }
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

template <class F, int MODE, class... As>
struct Engine {
    using Slots = cuda::std::tuple<Slot<As, MODE>...>;
    static constexpr int N = sizeof...(As);

    template <size_t... Is>
    __device__ __forceinline__ static void init_globals(Slots &s, const LaunchParams &p,
                                                        cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).init_global(p, int(Is)), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void init_elem(Slots &s, const LaunchParams &p, int64_t e,
                                                     char *smem, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).init_elem(p, int(Is), e, smem), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void init_elem_rec(Slots &s, const LaunchParams &p, int64_t e,
                                                         const int32_t *rk, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).init_elem_rec(p, int(Is), e, rk), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void init_tile(Slots &s, const LaunchParams &p, int64_t e,
                                                     const uint16_t *locs, char *const *gb, int U, int C,
                                                     cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).init_tile(p, int(Is), e, locs, gb, U, C), ...);
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
        if constexpr (((As::kind == KG && As::mode != MR) || ...)) {
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
    __device__ __forceinline__ static void zero_smem(Slots &s, const LaunchParams &p, int32_t b,
                                                     char *smem, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).zero_smem(p, int(Is), b, smem), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void write_back(Slots &s, const LaunchParams &p, int32_t b,
                                                      char *smem, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).write_back(p, int(Is), b, smem), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void backup_all(Slots &s, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).backup(), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void restore_all(Slots &s, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).restore(), ...);
    }
    // gather schedule, argument at position `a` among the mode-MM indirect args:
    // OP 0: run += its increments (INC); 1: its registers = run (WRITE, before
    // the call: the kernel sees the target's current value); 2: run = its registers
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
    // fold schedule: copy each INC argument's register increments into its
    // (position) slot of this element's shared-memory staging row
    template <int DGP, size_t... Is>
    __device__ __forceinline__ static void stage_incs(Slots &s, void *row,
                                                      cuda::std::index_sequence<Is...>) {
        (stage_inc_one<Is, DGP>(s, row), ...);
    }
    template <size_t I, int DGP>
    __device__ __forceinline__ static void stage_inc_one(Slots &s, void *row) {
        using A = cuda::std::tuple_element_t<I, cuda::std::tuple<As...>>;
        if constexpr (A::kind == KI && A::mode == MINC) {
            constexpr int pos = IncIndex<As...>::template of<I>();
            using T = typename A::type;
            T *dst = static_cast<T *>(row) + pos * DGP;
#pragma unroll
            for (int c = 0; c < A::dim; ++c) dst[c] = cuda::std::get<I>(s).acc[c];
        }
    }
    // tile gather: run += increments of the INC arguments on map column c
    template <int DG, class TG, size_t... Is>
    __device__ __forceinline__ static void gather_col(Slots &s, const LaunchParams &p, int c, TG *run,
                                                      cuda::std::index_sequence<Is...>) {
        (gather_col_one<Is, DG>(s, p, c, run), ...);
    }
    template <size_t I, int DG, class TG>
    __device__ __forceinline__ static void gather_col_one(Slots &s, const LaunchParams &p, int c, TG *run) {
        using A = cuda::std::tuple_element_t<I, cuda::std::tuple<As...>>;
        if constexpr (A::kind == KI && A::mode == MINC) {
            if (p.t.slot[I] == c) {
                auto &acc = cuda::std::get<I>(s).acc;
#pragma unroll
                for (int q = 0; q < DG; ++q) run[q] += acc[q];
            }
        }
    }
    // primary fold: READ args on the target's own column read its staged rows
    template <class TO, size_t... Is>
    __device__ __forceinline__ static void own_views(Slots &s, const LaunchParams &p, TO *own,
                                                     cuda::std::index_sequence<Is...>) {
        (own_view_one<Is>(s, p, own), ...);
    }
    template <size_t I, class TO>
    __device__ __forceinline__ static void own_view_one(Slots &s, const LaunchParams &p, TO *own) {
        using A = cuda::std::tuple_element_t<I, cuda::std::tuple<As...>>;
        if constexpr (A::kind == KI && A::mode == MR) {
            const int g = p.pf.own_grp[I];
            if (g >= 0) {
                using T = typename A::type;
                auto &sl = cuda::std::get<I>(s);
                sl.ptr = reinterpret_cast<T *>(own) + int64_t(p.pf.own_goff[g]) * blockDim.x;
                sl.sc = blockDim.x;
            }
        }
    }
    // primary fold: INC arguments at positions >= 1 -> the element's slots
    // slots: the element's secondary increments go to the rows of the targets'
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
    template <size_t... Is>
    __device__ __forceinline__ static void arrive_sums(Slots &s, const LaunchParams &p, int32_t b,
                                                       char *smem, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).arrive_sums(p, int(Is), b, smem), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void arrive_count(Slots &s, const LaunchParams &p, int32_t b,
                                                        char *smem, int *nfin,
                                                        cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).arrive_count(p, int(Is), b, smem, nfin), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void arrive_final(Slots &s, const LaunchParams &p, char *smem,
                                                        const int *nfin, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).arrive_final(p, int(Is), smem, nfin), ...);
    }
    template <size_t... Is>
    __device__ __forceinline__ static void apply_staged(Slots &s, cuda::std::index_sequence<Is...>) {
        (cuda::std::get<Is>(s).apply_staged(), ...);
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
};

template <class F, class... As>
__device__ __forceinline__ void run_direct(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_NONE, As...>;
    __shared__ double smem[32];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    typename E::Slots s;
    E::init_globals(s, p, idx);
    // persistent grid: CTA-strided over the plan blocks; one reduction
    // partial per CTA (folded in CTA order by k_combine)
    const int64_t nb = (p.n + p.bs - 1) / p.bs;
    for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int64_t lo = b * p.bs, hi = lo + p.bs < p.n ? lo + p.bs : p.n;
        for (int64_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
            E::init_elem(s, p, e, nullptr, idx);
            E::call(s, p, e, idx);
        }
    }
    if constexpr (E::has_reduce) E::reduce_all(s, p, blockIdx.x, smem, idx);
}

template <class F, class... As>
__device__ __forceinline__ void run_staged(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_REG, As...>;
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
        E::init_elem(s, p, e, nullptr, idx);
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

// Increments staged in shared memory: compute -> colour phases into smem ->
// one coalesced read-modify-write of the block's unique targets.
template <class F, int MODE, class... As>
__device__ __forceinline__ void run_smem(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, MODE, As...>;
    __shared__ double red[32];
    extern __shared__ __align__(16) char dsm[];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    const int32_t b = p.blocks[blockIdx.x];
    const int64_t e = int64_t(b) * p.bs + threadIdx.x;
    const int64_t hi = int64_t(b) * p.bs + p.bs < p.n ? int64_t(b) * p.bs + p.bs : p.n;
    const bool active = threadIdx.x < p.bs && e < hi;
    const int ncol = p.encol[b];
    const int mine = active ? int(p.ecol[e]) : -1;
    typename E::Slots s;
    if constexpr (MODE == ST_SMEM) E::zero_smem(s, p, b, dsm, idx);
    E::init_globals(s, p, idx);
    if (active) {
        E::init_elem(s, p, e, dsm, idx);
        E::call(s, p, e, idx);
    }
    __syncthreads();
    if constexpr (MODE == ST_SMEM) {
        for (int c = 0; c < ncol; ++c) {
            if (mine == c) E::apply_staged(s, idx);
            __syncthreads();
        }
    }
    E::write_back(s, p, b, dsm, idx);
    if constexpr (E::has_reduce) E::reduce_all(s, p, b, red, idx);
}

// Dataflow schedule: a persistent grid pulls blocks in plan (colour) order from
// a global counter.  Gather + compute + in-block colour phases run at once; the
// write-back waits only for the lower-colour blocks this block conflicts with,
// so colours overlap without grid-wide barriers while every target still sees
// its increments in exactly the order of the per-colour launch schedule.
// Polling uses relaxed gpu-scope loads: an acquire load would invalidate the
// whole L1 (CCTL.IVALL) on every spin, evicting the gathered data of every
// CTA on the SM.  The write-back reads its targets with ld.global.cg (L2, the
// coherence point), after the flag was observed and a CTA barrier, and the
// producer publishes with st.release after its CTA barrier — so the targets
// it wrote are visible in L2 before the flag is.
__device__ __forceinline__ int ld_relaxed(const int32_t *p) {
    int v;
    asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int32_t *p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

template <class F, int MODE, class... As>
__device__ __forceinline__ void run_flow(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, MODE, As...>;
    __shared__ double red[32];
    __shared__ int s_q;
    extern __shared__ __align__(16) char dsm[];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    int32_t *counter = p.flags + p.nqueue;
    if (threadIdx.x == 0) s_q = atomicAdd(counter, 1);
    __syncthreads();
    int q = s_q;
    while (q < p.nqueue) {
        // prefetch the next queue position while this block is processed
        int next = 0;
        if (threadIdx.x == 0) next = atomicAdd(counter, 1);
        const int32_t b = p.blocks[q];
        const int d0 = p.dep_off[b], d1 = p.dep_off[b + 1];
        const int32_t dep = d0 + int(threadIdx.x) < d1 ? p.dep_list[d0 + threadIdx.x] : -1;
        const int64_t e = int64_t(b) * p.bs + threadIdx.x;
        const int64_t hi = int64_t(b) * p.bs + p.bs < p.n ? int64_t(b) * p.bs + p.bs : p.n;
        const bool active = threadIdx.x < p.bs && e < hi;
        const int ncol = p.encol[b];
        const int mine = active ? int(p.ecol[e]) : -1;
        typename E::Slots s;
        if constexpr (MODE == ST_SMEM) E::zero_smem(s, p, b, dsm, idx);
        E::init_globals(s, p, idx);
        if (active) {
            E::init_elem(s, p, e, dsm, idx);
            E::call(s, p, e, idx);
        }
        __syncthreads();
        if constexpr (MODE == ST_SMEM) {
            for (int c = 0; c < ncol; ++c) {
                if (mine == c) E::apply_staged(s, idx);
                __syncthreads();
            }
        }
        // wait for the conflicting earlier-queued blocks (one thread per dependency)
        if (dep >= 0)
            while (ld_relaxed(p.flags + dep) == 0) __nanosleep(32);
        for (int k = d0 + int(threadIdx.x) + int(blockDim.x); k < d1; k += blockDim.x)
            while (ld_relaxed(p.flags + p.dep_list[k]) == 0) __nanosleep(32);
        __syncthreads();
        E::write_back(s, p, b, dsm, idx);
        if constexpr (E::has_reduce) E::reduce_all(s, p, b, red, idx);
        if (threadIdx.x == 0) s_q = next;
        __syncthreads();
        if (threadIdx.x == 0) st_release(p.flags + b, 1);
        q = s_q;
    }
}

// Target-centric ("gather") schedule for loops whose indirect writes all go to
// one dat with one mode — INC, or WRITE — and that write no direct argument: one
// thread per target element re-evaluates the kernel for every (element,
// argument) incidence of that target, in serial order, and keeps only that
// argument's effect on a running value that starts from the target's current
// value: INC adds the increment, WRITE replaces the value (the kernel is handed
// the running value in that argument, so it sees what the serial order would
// show it).  The target's final value is therefore exactly the serial one.  No
// colours, no shared memory, no atomics; a target's running value never leaves
// the thread's registers.  Global reductions count each element once (on its
// incidence through the first such argument).
template <class F, class... As>
__device__ __forceinline__ void run_gather(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_GATHER, As...>;
    constexpr bool has_inc = ((As::kind == KI && As::mode == MINC) || ...);
    constexpr int MM = has_inc ? MINC : MW;
    constexpr int G = ModeIndex<MM, As...>::template first<0>();
    static_assert(G >= 0, "gather schedule needs an INC or WRITE indirect argument");
    using AG = cuda::std::tuple_element_t<G, cuda::std::tuple<As...>>;
    using TG = typename AG::type;
    constexpr int DG = AG::dim;
    __shared__ double red[32];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    typename E::Slots s;
    E::init_globals(s, p, idx);
    // grid-stride over blocks of targets (a smaller grid keeps fewer targets'
    // rows in flight per SM; the default grid covers every target once)
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
         t - threadIdx.x < p.g_ntargets; t += int64_t(gridDim.x) * blockDim.x) {
        if (t >= p.g_ntargets) continue;
        const ArgRt &rg = p.a[G];
        const int64_t tg = p.g_tlist ? int64_t(__ldg(p.g_tlist + t)) : t;
        TG *dst = static_cast<TG *>(rg.data) + tg * rg.se;
        const int32_t seg = (MM == MINC && p.g_seg) ? __ldg(p.g_seg + t) : -1;
        TG run[DG];
#pragma unroll
        for (int c = 0; c < DG; ++c) run[c] = seg < 0 ? dst[c * rg.sc] : TG(0);
        for (int k = __ldg(p.g_off + t), ke = __ldg(p.g_off + t + 1); k < ke; ++k) {
            const int64_t e = __ldg(p.g_elem + k);
            const int a = __ldg(p.g_pos + k);
            E::init_elem(s, p, e, nullptr, idx);
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
            for (int c = 0; c < DG; ++c) dst[c * rg.sc] = run[c];
        }
    }
    if constexpr (E::has_reduce) E::reduce_all(s, p, blockIdx.x, red, idx);
}

// Hub targets of the gather schedule: value + the partial of each of its
// rows, in row (= element) order.
template <class T, int DG>
__global__ void __launch_bounds__(256) k_gather_hubs(const __grid_constant__ LaunchParams p, int ga) {
    pdl_wait();
    const int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (h >= p.g_nhub) return;
    const ArgRt &rg = p.a[ga];
    T *dst = static_cast<T *>(rg.data) + int64_t(__ldg(p.g_hub_tl + h)) * rg.se;
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

// Primary-fold schedule, pass 1 (see PFoldParams): a persistent grid strides
// over the targets; thread t evaluates, in element order, every element whose
// first INC argument targets it — each element exactly once in the whole
// launch, its neighbours' rows read once per element instead of once per
// incidence — adds that argument's increments to a running value that starts
// from the target's current value, and stores the other INC arguments'
// increments in the element's slots.  Global reductions count every element
// here (once).  Pass 2 (k_pfold_rest) adds each target's slots in element
// order.  Per target the result is value + primary increments + secondary
// increments: deterministic, within rounding of the serial order.
template <class TG, int DG>
struct PFoldShape {
    static constexpr int DGP = (DG + 1) / 2 * 2;   // slot rows of whole 16-byte pairs
};

template <class F, class... As>
__device__ __forceinline__ void run_pfold1(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_GATHER, As...>;
    constexpr int G = IncIndex<As...>::template first<0>();
    static_assert(G >= 0, "primary fold needs an INC argument");
    using AG = cuda::std::tuple_element_t<G, cuda::std::tuple<As...>>;
    using TG = typename AG::type;
    constexpr int DG = AG::dim;
    constexpr int NW = ((As::kind == KI && As::mode == MINC) + ...);
    constexpr int DGP = PFoldShape<TG, DG>::DGP;
    __shared__ double red[32];
    extern __shared__ __align__(16) char dsm[];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    typename E::Slots s;
    E::init_globals(s, p, idx);
    const PFoldParams &pf = p.pf;
    TG *own = reinterpret_cast<TG *>(dsm) + threadIdx.x;      // this thread's column
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t - threadIdx.x < pf.n1;
         t += int64_t(gridDim.x) * blockDim.x) {
        if (t >= pf.n1) continue;
        const ArgRt &rg = p.a[G];
        const int64_t tg = pf.tl1 ? int64_t(__ldg(pf.tl1 + t)) : t;
        TG *dst = static_cast<TG *>(rg.data) + tg * rg.se;
        const int32_t seg = pf.seg1 ? __ldg(pf.seg1 + t) : -1;
        // the target's own READ rows, once per target (consecutive targets: coalesced)
        for (int g = 0; g < pf.own_ngrp; ++g) {
            const ArgRt &r = p.a[pf.own_garg[g]];
            const TG *src = static_cast<const TG *>(r.data) + tg * r.se;
            TG *o = own + int64_t(pf.own_goff[g]) * blockDim.x;
            const int dim = pf.own_gdim[g];
#pragma unroll 4
            for (int c = 0; c < dim; ++c) o[c * blockDim.x] = __ldg(src + c * r.sc);
        }
        TG run[DG];
#pragma unroll
        for (int c = 0; c < DG; ++c) run[c] = seg < 0 ? dst[c * rg.sc] : TG(0);
        for (int k = __ldg(pf.off1 + t), ke = __ldg(pf.off1 + t + 1); k < ke; ++k) {
            const int64_t e = __ldg(pf.elem1 + k);
            if (pf.rec)
                E::init_elem_rec(s, p, e, pf.rec + int64_t(k) * pf.ncol, idx);
            else
                E::init_elem(s, p, e, nullptr, idx);
            if (pf.own_ngrp > 0) E::own_views(s, p, own, idx);
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
            for (int c = 0; c < DG; ++c) dst[c * rg.sc] = run[c];
        }
    }
    if constexpr (E::has_reduce) E::reduce_all(s, p, blockIdx.x, red, idx);
}

// Primary-fold schedule, pass 2: each target adds its slots in element order.
template <class T, int DG>
__global__ void __launch_bounds__(256) k_pfold_rest(const __grid_constant__ LaunchParams p, int ga) {
    pdl_wait();
    constexpr int DGP = PFoldShape<T, DG>::DGP;
    const PFoldParams &pf = p.pf;
    const ArgRt &rg = p.a[ga];
    const T *slots = static_cast<const T *>(pf.slots);
    for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < pf.n2;
         t += int64_t(gridDim.x) * blockDim.x) {
        const int64_t tg = pf.tl2 ? int64_t(__ldg(pf.tl2 + t)) : t;
        T *dst = static_cast<T *>(rg.data) + tg * rg.se;
        const int32_t seg = pf.seg2 ? __ldg(pf.seg2 + t) : -1;
        T run[DG];
#pragma unroll
        for (int c = 0; c < DG; ++c) run[c] = seg < 0 ? dst[c * rg.sc] : T(0);
        for (int k = __ldg(pf.off2 + t), ke = __ldg(pf.off2 + t + 1); k < ke; ++k) {
            const T *src = slots + int64_t(k) * DGP;        // rows in CSR order: contiguous per target
            if constexpr (DG % 2 == 0 && cuda::std::is_same_v<T, double>) {
#pragma unroll
                for (int c = 0; c < DG; c += 2) {
                    const double2 v = __ldcs(reinterpret_cast<const double2 *>(src + c));
                    run[c] += v.x;
                    run[c + 1] += v.y;
                }
            } else {
#pragma unroll
                for (int c = 0; c < DG; ++c) run[c] += __ldcs(src + c);
            }
        }
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

// Pass 2, warp-cooperative: a warp owns 32 consecutive pass-2 rows, whose
// slots are one contiguous range; the lanes copy it through shared memory in
// coalesced 16-byte chunks, then each lane adds its own rows in order — the
// same per-target arithmetic as k_pfold_rest, with full-sector DRAM reads.
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
            dst = static_cast<T *>(rg.data) + tg * rg.se;
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

// Hub targets of a split pass (pfold): value + each partial slot in order.
template <class T, int DG>
__global__ void __launch_bounds__(256) k_fold_parts(const __grid_constant__ LaunchParams p, int ga, int64_t nhub,
                                                    const int32_t *hub_tl, const int32_t *hub_off,
                                                    const void *parts) {
    pdl_wait();
    const int64_t h = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (h >= nhub) return;
    const ArgRt &rg = p.a[ga];
    T *dst = static_cast<T *>(rg.data) + int64_t(__ldg(hub_tl + h)) * rg.se;
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

// Fold schedule, pass 1 — every element evaluated exactly once, like a direct
// loop (coalesced direct access, no colours): its INC increments, computed
// from zero in registers, go to the element's slots of an element-major
// buffer [n][INC args][DGP] (DGP = dim rounded up to 4 doubles, so a slot is
// whole 32-byte sectors) instead of the targets.  The slots of a CTA's 256
// elements are one contiguous region: they are staged through shared memory
// (rows padded by one word against bank conflicts) and stored coalesced.
// Pass 2 (k_fold_targets) adds each target's slots onto it in serial order.
// The increments are the very values the serial run adds (same functor, same
// zero start), added in the same order, so the result is the serial one bit
// for bit — with the kernel evaluated once per element instead of once per
// incidence as in the gather schedule.
template <class T, int DG>
struct FoldShape {
    static constexpr int DGP = (DG + 3) / 4 * 4;
};

template <class F, class... As>
__device__ __forceinline__ void run_fold_edges(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_REG, As...>;
    constexpr int G = IncIndex<As...>::template first<0>();
    using AG = cuda::std::tuple_element_t<G, cuda::std::tuple<As...>>;
    using TG = typename AG::type;
    constexpr int NW = ((As::kind == KI && As::mode == MINC) + ...);
    constexpr int DGP = FoldShape<TG, AG::dim>::DGP;
    constexpr int ROW = NW * DGP, SROW = ROW + 1;
    __shared__ double red[32];
    extern __shared__ __align__(16) char dsm[];
    TG *st = reinterpret_cast<TG *>(dsm);
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    const int64_t e0 = int64_t(blockIdx.x) * blockDim.x, e = e0 + threadIdx.x;
    typename E::Slots s;
    E::init_globals(s, p, idx);
    if (e < p.n) {
        E::init_elem(s, p, e, nullptr, idx);
        E::call(s, p, e, idx);
        E::template stage_incs<DGP>(s, st + threadIdx.x * SROW, idx);
    }
    __syncthreads();
    const int64_t rows = p.n - e0 < int64_t(blockDim.x) ? p.n - e0 : int64_t(blockDim.x);
    TG *out = static_cast<TG *>(p.g_buf) + e0 * ROW;
    for (int k = threadIdx.x; k < rows * ROW; k += blockDim.x) {
        const int r = k / ROW, c = k - r * ROW;
        if (c % DGP < AG::dim) __stcg(out + k, st[r * SROW + c]);
    }
    if constexpr (E::has_reduce) E::reduce_all(s, p, blockIdx.x, red, idx);
}

template <class S>
struct FoldSmem;
template <class... As>
struct FoldSmem<Sig<As...>> {
    static size_t bytes(int threads) {
        constexpr int G = IncIndex<As...>::template first<0>() < 0 ? 0 : IncIndex<As...>::template first<0>();
        using AG = cuda::std::tuple_element_t<G, cuda::std::tuple<As...>>;
        constexpr int NW = ((As::kind == KI && As::mode == MINC) + ...);
        constexpr int DGP = FoldShape<typename AG::type, AG::dim>::DGP;
        return size_t(threads) * (NW * DGP + 1) * sizeof(typename AG::type);
    }
};

// Fold schedule, pass 2: one thread per target, slots in serial order.
template <class T, int DG>
__global__ void __launch_bounds__(256) k_fold_targets(const __grid_constant__ LaunchParams p, int ga) {
    constexpr int DGP = FoldShape<T, DG>::DGP;
    const int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= p.g_ntargets) return;
    const ArgRt &rg = p.a[ga];
    const int64_t tg = p.g_tlist ? int64_t(__ldg(p.g_tlist + t)) : t;
    T *dst = static_cast<T *>(rg.data) + tg * rg.se;
    const T *buf = static_cast<const T *>(p.g_buf);
    const int64_t row = int64_t(p.g_nw) * DGP;
    T run[DG];
#pragma unroll
    for (int c = 0; c < DG; ++c) run[c] = dst[c * rg.sc];
    for (int k = __ldg(p.g_off + t), ke = __ldg(p.g_off + t + 1); k < ke; ++k) {
        const T *src = buf + int64_t(__ldg(p.g_elem + k)) * row + int(__ldg(p.g_pos + k)) * DGP;
        if constexpr (DG % 2 == 0 && cuda::std::is_same_v<T, double>) {
#pragma unroll
            for (int c = 0; c < DG; c += 2) {   // 16-byte loads: slots are 32-byte aligned
                const double2 v = __ldcs(reinterpret_cast<const double2 *>(src + c));
                run[c] += v.x;
                run[c + 1] += v.y;
            }
        } else {
#pragma unroll
            for (int c = 0; c < DG; ++c) run[c] += __ldcs(src + c);
        }
    }
#pragma unroll
    for (int c = 0; c < DG; ++c) dst[c * rg.sc] = run[c];
}

// Tile schedule (see host_tile.cpp): one CTA per tile.
//  1. stage: the tile's target list, then every READ dat's rows of the staged
//     targets, copied HBM/L2 -> shared memory with cp.async (8-byte copies,
//     no registers held, thousands in flight per CTA), component-major
//     [dim][U]; INC accumulators of the owned targets [dim][C] zeroed;
//  2. evaluate: the tile's elements in chunks of blockDim; READ args are
//     shared-memory views, direct args HBM views, INC args registers;
//  3. apply: element-colour phases add the register increments of owned
//     targets into the accumulators (elements of one colour share no owned
//     target), so no atomics and a fixed order — deterministic run to run;
//  4. write back: one read-modify-write per owned target and component.
// A target's increments all come from its owning tile, so tiles never
// conflict: one launch, no block colours, no inter-CTA synchronisation.
__device__ __forceinline__ void cp_async8(void *smem_dst, const void *gsrc) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

template <class S>
struct TileType;
template <class... As>
struct TileType<Sig<As...>> {
    static constexpr int G = IncIndex<As...>::template first<0>() < 0 ? 0 : IncIndex<As...>::template first<0>();
    using type = typename cuda::std::tuple_element_t<G, cuda::std::tuple<As...>>::type;
};

__host__ __device__ inline size_t tile_align(size_t x) { return (x + 15) / 16 * 16; }

template <class F, class... As>
__device__ __forceinline__ void run_tile(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_TILE, As...>;
    using T = typename TileType<Sig<As...>>::type;
    __shared__ double red[32];
    extern __shared__ __align__(16) char dsm[];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    const TileParams &tp = p.t;
    const int32_t t = blockIdx.x;
    const int32_t l0 = tp.list_off[t], U = tp.list_off[t + 1] - l0, C = tp.nown[t];
    const int ng = tp.nread + tp.ninc;
#ifdef ML_TILE_PROFILE
    long long tk0 = clock64(), tk1 = 0, tk2 = 0, tk3 = 0, tk4 = 0;
#endif
    int32_t *slist = reinterpret_cast<int32_t *>(dsm);
    __shared__ char *gb[MAX_TGROUPS];        // group bases (shared: indexed at run time)
    if (threadIdx.x == 0) {
        size_t off = tile_align(size_t(U) * 4);
        for (int g = 0; g < ng; ++g) {
            gb[g] = dsm + off;
            off += tile_align(sizeof(T) * size_t(tp.gdim[g]) * size_t(g < tp.nread ? U : C));
        }
    }
    __syncthreads();
    for (int g = tp.nread; g < ng; ++g) {
        T *acc = reinterpret_cast<T *>(gb[g]);
        for (int k = threadIdx.x; k < tp.gdim[g] * C; k += blockDim.x) acc[k] = T(0);
    }
    // one staged target per thread and pass: its id is loaded once, then every
    // component of every READ dat is copied (lanes = consecutive list entries)
    for (int j = threadIdx.x; j < U; j += blockDim.x) {
        const int64_t v = __ldg(tp.list + l0 + j);
        slist[j] = int32_t(v);
        for (int g = 0; g < tp.nread; ++g) {
            const ArgRt &r = p.a[tp.garg[g]];
            const T *src = static_cast<const T *>(r.data) + v * r.se;
            T *dst = reinterpret_cast<T *>(gb[g]) + j;
            const int dim = tp.gdim[g];
#pragma unroll 4
            for (int c = 0; c < dim; ++c) cp_async8(dst + c * U, src + c * r.sc);
        }
    }
#ifdef ML_TILE_PROFILE
    tk1 = clock64();
#endif
    cp_async_wait_all();
    __syncthreads();
#ifdef ML_TILE_PROFILE
    tk2 = clock64();
#endif

    typename E::Slots s;
    E::init_globals(s, p, idx);
    const int32_t k1 = tp.elem_off[t + 1];
    const int ncol = tp.ncol[t];
    for (int32_t k0 = tp.elem_off[t]; k0 < k1; k0 += blockDim.x) {
        const int32_t k = k0 + threadIdx.x;
        int mine = -1;
        if (k < k1) {
            const int64_t e = __ldg(tp.elem + k);
            const uint8_t fl = __ldg(tp.ecol + k);
            mine = fl & 127;
            E::init_tile(s, p, e, tp.loc + int64_t(k) * tp.arity, gb, U, C, idx);
            if constexpr (E::has_reduce) {
                if (!(fl & 128) || e >= p.rlim) {
                    E::backup_all(s, idx);
                    E::call_raw(s, p, idx);
                    E::restore_all(s, idx);
                } else {
                    E::call_raw(s, p, idx);
                }
            } else {
                E::call_raw(s, p, idx);
            }
        }
        for (int c = 0; c < ncol; ++c) {
            if (mine == c) E::apply_staged(s, idx);
            __syncthreads();
        }
    }
#ifdef ML_TILE_PROFILE
    tk3 = clock64();
#endif
    // write back: 4 independent read-modify-writes in flight per thread
    for (int g = tp.nread; g < ng; ++g) {
        const ArgRt &r = p.a[tp.garg[g]];
        T *d = static_cast<T *>(r.data);
        const T *acc = reinterpret_cast<const T *>(gb[g]);
        const int total = tp.gdim[g] * C;
        constexpr int UN = 4;
        for (int k0 = threadIdx.x; k0 < total; k0 += UN * blockDim.x) {
            int64_t a[UN];
            T v[UN];
#pragma unroll
            for (int q = 0; q < UN; ++q) {
                const int k = k0 + q * blockDim.x;
                if (k < total) {
                    const int c = k / C, j = k - c * C;
                    a[q] = int64_t(slist[j]) * r.se + c * r.sc;
                    v[q] = d[a[q]];
                }
            }
#pragma unroll
            for (int q = 0; q < UN; ++q)
                if (k0 + q * blockDim.x < total) d[a[q]] = v[q] + acc[k0 + q * blockDim.x];
        }
    }
#ifdef ML_TILE_PROFILE
    __syncthreads();
    tk4 = clock64();
    if (threadIdx.x == 0 && p.g_buf) {
        long long *o = static_cast<long long *>(p.g_buf) + int64_t(t) * 4;
        o[0] = tk1 - tk0; o[1] = tk2 - tk1; o[2] = tk3 - tk2; o[3] = tk4 - tk3;
    }
#endif
    if constexpr (E::has_reduce) E::reduce_all(s, p, t, red, idx);
}

// Tile-gather variant: the tile's staged rows as in run_tile, then one thread
// per owned target re-evaluates each of its incidences (element order, then
// column) from shared memory and keeps its own increments in registers — no
// colour phases, no accumulators, one barrier.  Elements are evaluated once
// per incidence (like the gather schedule) but every node row comes from
// shared memory, staged once per tile.  Reductions count an element at its
// `red_col` incidence (exactly one tile owns that target).
template <class F, class... As>
__device__ __forceinline__ void run_tgather(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_TILE, As...>;
    constexpr int G = IncIndex<As...>::template first<0>();
    using AG = cuda::std::tuple_element_t<G, cuda::std::tuple<As...>>;
    using T = typename AG::type;
    constexpr int DG = AG::dim;
    __shared__ double red[32];
    __shared__ char *gb[MAX_TGROUPS];
    extern __shared__ __align__(16) char dsm[];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    const TileParams &tp = p.t;
    const int32_t t = blockIdx.x;
    const int32_t l0 = tp.list_off[t], U = tp.list_off[t + 1] - l0, C = tp.nown[t];
    const int ng = tp.nread;
    int32_t *slist = reinterpret_cast<int32_t *>(dsm);
    if (threadIdx.x == 0) {
        size_t off = tile_align(size_t(U) * 4);
        for (int g = 0; g < ng; ++g) {
            gb[g] = dsm + off;
            off += tile_align(sizeof(T) * size_t(tp.gdim[g]) * size_t(U));
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < U; j += blockDim.x) {
        const int64_t v = __ldg(tp.list + l0 + j);
        slist[j] = int32_t(v);
        for (int g = 0; g < ng; ++g) {
            const ArgRt &r = p.a[tp.garg[g]];
            const T *src = static_cast<const T *>(r.data) + v * r.se;
            T *dst = reinterpret_cast<T *>(gb[g]) + j;
            const int dim = tp.gdim[g];
#pragma unroll 4
            for (int c = 0; c < dim; ++c) cp_async8(dst + c * U, src + c * r.sc);
        }
    }
    cp_async_wait_all();
    __syncthreads();
    typename E::Slots s;
    E::init_globals(s, p, idx);
    const int32_t e0 = tp.elem_off[t];
    const int32_t *ioff = tp.inc_off + tp.inc_base[t];
    const ArgRt &rg = p.a[G];
    for (int j = threadIdx.x; j < C; j += blockDim.x) {
        T *dst = static_cast<T *>(rg.data) + int64_t(slist[j]) * rg.se;
        T run[DG];
#pragma unroll
        for (int c = 0; c < DG; ++c) run[c] = dst[c * rg.sc];
        for (int q = __ldg(ioff + j), qe = __ldg(ioff + j + 1); q < qe; ++q) {
            const int k = e0 + __ldg(tp.inc_k + q);
            const int col = __ldg(tp.inc_c + q);
            const int64_t e = __ldg(tp.elem + k);
            E::init_tile(s, p, e, tp.loc + int64_t(k) * tp.arity, gb, U, 0, idx);
            if constexpr (E::has_reduce) {
                if (col != tp.red_col || e >= p.rlim) {
                    E::backup_all(s, idx);
                    E::call_raw(s, p, idx);
                    E::restore_all(s, idx);
                } else {
                    E::call_raw(s, p, idx);
                }
            } else {
                E::call_raw(s, p, idx);
            }
            E::template gather_col<DG>(s, p, col, run, idx);
        }
#pragma unroll
        for (int c = 0; c < DG; ++c) dst[c * rg.sc] = run[c];
    }
    if constexpr (E::has_reduce) E::reduce_all(s, p, t, red, idx);
}

// Arrival schedule: one launch over the plan blocks in natural order (best
// locality), no block colours and no inter-block waiting.  Targets touched by
// one block are updated directly; shared targets are completed by whichever
// block arrives last, folding the per-block partials in block order, so the
// result is deterministic run to run.  Partials of neighbouring blocks are
// written and read within a short time window, so they live in L2.
template <class F, class... As>
__device__ __forceinline__ void run_arrive(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_SEG, As...>;
    __shared__ double red[32];
    __shared__ int nfin[MAX_GROUPS];
    extern __shared__ __align__(16) char dsm[];
    constexpr auto idx = cuda::std::make_index_sequence<E::N>{};
    const int32_t b = blockIdx.x;
    const int64_t e = int64_t(b) * p.bs + threadIdx.x;
    const int64_t hi = int64_t(b) * p.bs + p.bs < p.n ? int64_t(b) * p.bs + p.bs : p.n;
    const bool active = threadIdx.x < p.bs && e < hi;
    if (threadIdx.x < MAX_GROUPS) nfin[threadIdx.x] = 0;
    typename E::Slots s;
    E::init_globals(s, p, idx);
    if (active) {
        E::init_elem(s, p, e, dsm, idx);
        E::call(s, p, e, idx);
    }
    __syncthreads();
    E::arrive_sums(s, p, b, dsm, idx);
    __threadfence();
    __syncthreads();
    E::arrive_count(s, p, b, dsm, nfin, idx);
    __syncthreads();
    E::arrive_final(s, p, dsm, nfin, idx);
    if constexpr (E::has_reduce) E::reduce_all(s, p, b, red, idx);
}

template <class F, class... As>
__device__ __forceinline__ void run_phased(const LaunchParams &p, Sig<As...>) {
    using E = Engine<F, ST_NONE, As...>;
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
            E::init_elem(s, p, e, nullptr, idx);
            E::call(s, p, e, idx);
        }
        __syncthreads();
    }
    if constexpr (E::has_reduce) E::reduce_all(s, p, b, smem, idx);
}

template <class F, class T>
__global__ void __launch_bounds__(256) k_direct(const __grid_constant__ LaunchParams p) {
    pdl_wait();
    run_direct<F>(p, typename F::template sig<T>{});
}
template <class F, class T>
__global__ void __launch_bounds__(256) k_staged(const __grid_constant__ LaunchParams p) {
    run_staged<F>(p, typename F::template sig<T>{});
}
template <class F, class T>
__global__ void __launch_bounds__(256) k_phased(const __grid_constant__ LaunchParams p) {
    run_phased<F>(p, typename F::template sig<T>{});
}
template <class F, class T, int MODE>
__global__ void __launch_bounds__(256) k_smem(const __grid_constant__ LaunchParams p) {
    run_smem<F, MODE>(p, typename F::template sig<T>{});
}
template <class F, class T, int MODE>
__global__ void __launch_bounds__(256) k_flow(const __grid_constant__ LaunchParams p) {
    run_flow<F, MODE>(p, typename F::template sig<T>{});
}
template <class F, class T>
__global__ void __launch_bounds__(256) k_fold_edges(const __grid_constant__ LaunchParams p) {
    run_fold_edges<F>(p, typename F::template sig<T>{});
}
template <class F, class T>
__global__ void __launch_bounds__(256) k_arrive(const __grid_constant__ LaunchParams p) {
    run_arrive<F>(p, typename F::template sig<T>{});
}
template <class F, class T, int NT>
__global__ void __launch_bounds__(NT, 512 / NT) k_tile(const __grid_constant__ LaunchParams p) {
    run_tile<F>(p, typename F::template sig<T>{});
}
template <class F, class T, int NT>
__global__ void __launch_bounds__(NT, 512 / NT) k_tgather(const __grid_constant__ LaunchParams p) {
    run_tgather<F>(p, typename F::template sig<T>{});
}
template <class F, class T>
__global__ void __launch_bounds__(256) k_pfold1(const __grid_constant__ LaunchParams p) {
    pdl_wait();
    run_pfold1<F>(p, typename F::template sig<T>{});
}
template <class F, class T>
__global__ void __launch_bounds__(256) k_gather(const __grid_constant__ LaunchParams p) {
    pdl_wait();
    run_gather<F>(p, typename F::template sig<T>{});
}
template <class F, class T, int MINB>
__global__ void __launch_bounds__(256, MINB) k_gather_occ(const __grid_constant__ LaunchParams p) {
    run_gather<F>(p, typename F::template sig<T>{});
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
    // fold schedule: indirect writes all INC (direct writes allowed)
    static constexpr bool fold_ok = ind_inc && !ind_rw && !ind_w;
    // tile schedule: indirect writes all INC, no direct writes (cut elements
    // are evaluated by two tiles)
    static constexpr bool tile_ok = ind_inc && !ind_rw && !ind_w && !direct_write;
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
    LaunchFn direct, staged, phased;
    LaunchFn smem[2], flow[2];                       // [0] colour phases, [1] segmented
    LaunchFn arrive;                                 // segmented, no block colours
    LaunchFn gather[4];                              // target-centric (INC-only or WRITE-only):
                                                     // free / >=2 / >=3 / >=4 CTAs of 256 per SM
    int (*flow_occupancy[2])(int threads, size_t smem);
    int (*gather_occupancy)();
    int (*direct_occupancy)(int threads);
    LaunchFn fold_edges, fold_targets;               // fold schedule (INC-only indirect writes)
    int32_t fold_dim, fold_arg;                      // INC dim, first INC argument
    LaunchFn tile;                                   // tile schedule (INC-only, no direct writes)
    LaunchFn tgather;                                // tile-gather variant
    LaunchFn pfold1, pfold2;                         // primary-fold schedule (INC-only)
    LaunchFn gather_hubs;                            // hub fix-up of the gather schedule (INC)
    int (*pfold_occupancy)(size_t smem);
    void (*pfold_hubs)(const LaunchParams &, int64_t nhub, const int32_t *tl, const int32_t *off,
                       const void *parts, cudaStream_t);
    int32_t pfold_dgp, pfold_nslot;
};

void register_functor(const FunctorEntry &e);

template <class F, class T>
struct Registrar {
    static void direct(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        launch_k(k_direct<F, T>, g, b, 0, s, p);
    }
    static int direct_occupancy(int threads) {
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_direct<F, T>, threads, 0) != cudaSuccess) n = 0;
        return n;
    }
    static void staged(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        k_staged<F, T><<<g, b, 0, s>>>(p);
    }
    static void phased(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        k_phased<F, T><<<g, b, 0, s>>>(p);
    }
    template <int MODE>
    static void smem(const LaunchParams &p, dim3 g, dim3 b, size_t bytes, cudaStream_t s) {
        static bool opted = false;
        if (!opted && bytes > 48 * 1024) {
            cudaFuncSetAttribute(k_smem<F, T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            opted = true;
        }
        k_smem<F, T, MODE><<<g, b, bytes, s>>>(p);
    }
    template <int MODE>
    static void flow(const LaunchParams &p, dim3 g, dim3 b, size_t bytes, cudaStream_t s) {
        static bool opted = false;
        if (!opted && bytes > 48 * 1024) {
            cudaFuncSetAttribute(k_flow<F, T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            opted = true;
        }
        k_flow<F, T, MODE><<<g, b, bytes, s>>>(p);
    }
    static void gather(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        static bool once = false;
        if (!once) {   // no shared memory to speak of: give the SM's storage to L1
            cudaFuncSetAttribute(k_gather<F, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
            once = true;
        }
        launch_k(k_gather<F, T>, g, b, 0, s, p);
    }
    // resident CTAs of 256 threads per SM (sizes the persistent gather grid)
    static int gather_occupancy() {
        static int n = -1;
        if (n < 0) {
            cudaFuncSetAttribute(k_gather<F, T>, cudaFuncAttributePreferredSharedMemoryCarveout, 0);
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_gather<F, T>, 256, 0) != cudaSuccess) n = 0;
        }
        return n;
    }
    static void fold_edges(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        using S = typename F::template sig<T>;
        const size_t bytes = FoldSmem<S>::bytes(int(b.x));
        static bool once = false;
        if (!once) {
            if (bytes > 48 * 1024)
                cudaFuncSetAttribute(k_fold_edges<F, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            once = true;
        }
        k_fold_edges<F, T><<<g, b, bytes, s>>>(p);
    }
    static void gather_hubs(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        using S = typename F::template sig<T>;
        using AG = typename FirstInc<S>::type;
        launch_k(k_gather_hubs<typename AG::type, AG::dim>, g, b, 0, s, p, int(FirstInc<S>::value));
    }
    static void pfold_attrs(size_t bytes) {
        static int carve = -1;
        const int want = bytes ? 100 : 0;
        if (carve != want) {
            cudaFuncSetAttribute(k_pfold1<F, T>, cudaFuncAttributePreferredSharedMemoryCarveout, want);
            carve = want;
        }
        static size_t opted = 48 * 1024;
        if (bytes > opted) {
            cudaFuncSetAttribute(k_pfold1<F, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
            opted = bytes;
        }
    }
    static void pfold1(const LaunchParams &p, dim3 g, dim3 b, size_t bytes, cudaStream_t s) {
        pfold_attrs(bytes);
        launch_k(k_pfold1<F, T>, g, b, bytes, s, p);
    }
    static int pfold_occupancy(size_t bytes) {
        pfold_attrs(bytes);
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_pfold1<F, T>, 256, bytes) != cudaSuccess) n = 0;
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
        if (pass2_warp())
            launch_k(k_pfold_rest_w<typename AG::type, AG::dim>, g, b, 0, s, p, int(FirstInc<S>::value));
        else
            launch_k(k_pfold_rest<typename AG::type, AG::dim>, g, b, 0, s, p, int(FirstInc<S>::value));
    }
    static void fold_targets(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        using S = typename F::template sig<T>;
        constexpr int G = FirstInc<S>::value;
        using AG = typename FirstInc<S>::type;
        k_fold_targets<typename AG::type, AG::dim><<<g, b, 0, s>>>(p, G);
    }
    template <int NT>
    static void tile_launch(const LaunchParams &p, dim3 g, size_t bytes, cudaStream_t s) {
        static size_t opted = 48 * 1024;
        if (bytes > opted) {
            cudaFuncSetAttribute(k_tile<F, T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
            opted = bytes;
        }
        k_tile<F, T, NT><<<g, NT, bytes, s>>>(p);
    }
    template <int NT>
    static void tgather_launch(const LaunchParams &p, dim3 g, size_t bytes, cudaStream_t s) {
        static size_t opted = 48 * 1024;
        if (bytes > opted) {
            cudaFuncSetAttribute(k_tgather<F, T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
            opted = bytes;
        }
        k_tgather<F, T, NT><<<g, NT, bytes, s>>>(p);
    }
    static void tgather(const LaunchParams &p, dim3 g, dim3 b, size_t bytes, cudaStream_t s) {
        if (b.x == 128) tgather_launch<128>(p, g, bytes, s);
        else tgather_launch<256>(p, g, bytes, s);
    }
    static void tile(const LaunchParams &p, dim3 g, dim3 b, size_t bytes, cudaStream_t s) {
        if (b.x == 128) tile_launch<128>(p, g, bytes, s);
        else tile_launch<256>(p, g, bytes, s);
    }
    template <int MINB>
    static void gather_occ(const LaunchParams &p, dim3 g, dim3 b, size_t, cudaStream_t s) {
        k_gather_occ<F, T, MINB><<<g, b, 0, s>>>(p);
    }
    static void arrive(const LaunchParams &p, dim3 g, dim3 b, size_t bytes, cudaStream_t s) {
        static bool opted = false;
        if (!opted && bytes > 48 * 1024) {
            cudaFuncSetAttribute(k_arrive<F, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
            opted = true;
        }
        k_arrive<F, T><<<g, b, bytes, s>>>(p);
    }
    template <int MODE>
    static int flow_occupancy(int threads, size_t bytes) {
        if (bytes > 48 * 1024)
            cudaFuncSetAttribute(k_flow<F, T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        int n = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, k_flow<F, T, MODE>, threads, bytes) != cudaSuccess)
            return 0;
        return n;
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
        e.direct = &direct;
        e.direct_occupancy = &direct_occupancy;
        e.staged = SigInfo<S>::ind_write && !SigInfo<S>::ind_write_non_inc ? &staged : nullptr;
        e.phased = SigInfo<S>::ind_write ? &phased : nullptr;
        const bool st = e.staged != nullptr;
        e.smem[0] = st ? &smem<ST_SMEM> : nullptr;
        e.smem[1] = st ? &smem<ST_SEG> : nullptr;
        e.flow[0] = st ? &flow<ST_SMEM> : nullptr;
        e.flow[1] = st ? &flow<ST_SEG> : nullptr;
        e.flow_occupancy[0] = st ? &flow_occupancy<ST_SMEM> : nullptr;
        e.flow_occupancy[1] = st ? &flow_occupancy<ST_SEG> : nullptr;
        e.arrive = st ? &arrive : nullptr;
        if constexpr (SigInfo<S>::fold_ok) {
            e.pfold1 = &pfold1;
            e.pfold2 = &pfold2;
            e.pfold_occupancy = &pfold_occupancy;
            e.pfold_hubs = &pfold_hubs;
            using AG = typename FirstInc<S>::type;
            e.pfold_dgp = PFoldShape<typename AG::type, AG::dim>::DGP;
            e.pfold_nslot = SigInfo<S>::n_inc - 1;
            e.fold_edges = &fold_edges;
            e.fold_targets = &fold_targets;
            e.fold_arg = FirstInc<S>::value;
            e.fold_dim = FirstInc<S>::type::dim;
        }
        if constexpr (SigInfo<S>::tile_ok) {
            e.tile = &tile;
            e.tgather = &tgather;
        }
        if constexpr (SigInfo<S>::gather_ok && SigInfo<S>::ind_inc) e.gather_hubs = &gather_hubs;
        if constexpr (SigInfo<S>::gather_ok) {
            e.gather_occupancy = &gather_occupancy;
            e.gather[0] = &gather;
            e.gather[1] = &gather_occ<2>;
            e.gather[2] = &gather_occ<3>;
            e.gather[3] = &gather_occ<4>;
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
