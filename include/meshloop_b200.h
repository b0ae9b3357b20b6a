/*
 * meshloop_b200.h — C ABI of libmeshloop_b200.so, the B200 execution backend
 * for the OP2-style op_par_loop abstraction of arXiv:1403.7209.
 *
 * The reference (`meshloop`, pure Python + numpy, /root/reference/pkg) has no
 * FFI: its "plugin interface" for this path is the loop descriptor + kernel
 * callback contract and the closed backend switch of run_program.  Each entry
 * point below replaces one reference function on the hot path; the citation
 * is `pkg/src/meshloop/<file>:<line>`.  INTEGRATION.md shows the ctypes stub
 * a maintainer would add to meshloop to bind them.
 *
 * Conventions
 *   - every function returns 0 on success or a negative ML_E* code; the
 *     message is available from ml_last_error() (thread-local);
 *   - no C++ exceptions cross the ABI; plain pointers and sizes only;
 *   - host pointers are borrowed for the duration of a call;
 *   - device memory is owned by the library (ml_alloc/ml_free);
 *   - all device work is enqueued on the library's compute stream of the
 *     current device; ml_synchronize() waits for it.
 */
#ifndef MESHLOOP_B200_H
#define MESHLOOP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- error codes -------------------------------------------------------- */
#define ML_OK          0
#define ML_EINVAL     -1   /* bad argument / signature mismatch             */
#define ML_ECUDA      -2   /* CUDA runtime error                            */
#define ML_ENOMEM     -3   /* allocation failed                             */
#define ML_ENOFUNCTOR -4   /* no compiled functor of that name/dtype        */
#define ML_ENCCL      -5   /* NCCL error / exchange timeout                 */

/* ---- argument descriptors (core.py:223-254, 50-71) ----------------------- */
enum { ML_DIRECT = 0, ML_INDIRECT = 1, ML_GLOBAL = 2 };
enum { ML_READ = 0, ML_WRITE = 1, ML_RW = 2, ML_INC = 3, ML_MIN = 4, ML_MAX = 5 };
enum { ML_F64 = 0, ML_I64 = 1 };
enum { ML_AOS = 0, ML_SOA = 1 };

typedef struct ml_arg {
    int32_t kind;          /* ML_DIRECT / ML_INDIRECT / ML_GLOBAL                 */
    int32_t mode;          /* ML_READ .. ML_MAX                                   */
    int32_t dim;           /* components per element (global: buffer length)      */
    int32_t dtype;         /* ML_F64 / ML_I64                                     */
    int32_t layout;        /* ML_AOS / ML_SOA (dat args)                          */
    int32_t slot;          /* 0-based map column (indirect args)                  */
    void *data;            /* device payload of the dat, or device global buffer  */
    const int32_t *map;    /* device map table, column-major int32 [arity][from]  */
    int64_t map_from;      /* from-set size of the map (column stride)            */
    int64_t set_size;      /* size of the dat's set                               */
    int64_t pitch;         /* plain SOA (seg_shift 0): component stride in elements
                              of the device copy (>= set_size; 0 means set_size) */
    int32_t seg_shift;     /* segmented SOA: the device copy stores segments of
                              2^s elements, each segment's components one after
                              another at stride P = 2^s + ML_SEG_PAD: (e, c) at
                              (e >> s) * P * dim + c * P + (e & (2^s - 1)).  The
                              library's own SOA copies use s = ML_SEG_SHIFT;
                              0: plain SOA                                     */
} ml_arg_t;
#ifndef ML_SEG_SHIFT
#define ML_SEG_SHIFT 6
#endif
#ifndef ML_SEG_PAD
#define ML_SEG_PAD 0
#endif
/* SOA dats of dim ML_SEG_MIN_DIM..ML_SEG_MAX_DIM are segmented on the device
 * (AoSoA: blocks of 2^ML_SEG_SHIFT elements, each holding its components one
 * after another); other SOA dats keep plain component rows padded to 32
 * elements.  Default: the wide dats (>= 8 components) in 64-element blocks —
 * on the Hydra proxy the fused flux loop gathers lim/grad/aux 6 % faster and
 * nothing else moves; segmenting the 6-component dats too, or padding the
 * blocks, is slower (profiles/r2/seg_sweep.md).  Host copies go through a
 * device repack kernel (ml_seg_copy), so they run at full PCIe speed. */
#ifndef ML_SEG_MAX_DIM
#define ML_SEG_MAX_DIM 64
#endif
#ifndef ML_SEG_MIN_DIM
#define ML_SEG_MIN_DIM 8
#endif

/* Device copy of an execution plan (plan.py:30-45).  `color_offsets` is a
 * HOST array; the rest are device arrays produced by ml_plan_* below. */
typedef struct ml_plan_dev {
    int64_t nblocks;
    int64_t ncolors;
    int64_t block_size;
    const int64_t *color_offsets;   /* host [ncolors+1] into `blocks`           */
    const int32_t *blocks;          /* device: block ids ordered by colour      */
    const uint16_t *elem_color;     /* device [n]; NULL when no indirect writes */
    const int32_t *elem_ncolors;    /* device [nblocks]; NULL likewise          */
} ml_plan_dev_t;

#define ML_MAX_ARGS 16

typedef struct ml_loop {
    const char *name;               /* for error messages                       */
    int32_t functor;                /* id from ml_functor_lookup                */
    int32_t nargs;
    const ml_arg_t *args;
    int64_t n;                      /* iteration-set size                       */
    ml_plan_dev_t plan;
    double fconst[4];               /* kernel constants (e.g. dt)               */
    int64_t iconst[4];              /* kernel constants (e.g. integer scale)    */
    void *scratch;                  /* device scratch >= ml_loop_scratch_bytes,
                                       zero-filled when allocated               */
    int64_t rlim;                   /* elements >= rlim skip global reductions
                                       (exec-halo elements on multi-GPU runs);
                                       < 0 means n                               */
    /* target-centric schedule (ml_gather_build); ntargets == 0 disables it */
    int64_t gather_ntargets;
    const int32_t *gather_off;      /* device [ntargets+1]                       */
    const int32_t *gather_elem;     /* device [n * written args]                 */
    const uint8_t *gather_pos;      /* device [n * written args]                 */
    const int32_t *gather_targets;  /* device [ntargets] target ids of a compacted
                                       list (only targets with incidences), or
                                       NULL: target k is element k of the set   */
    /* hub splitting (INC gather only; gather_seg NULL disables it): rows of
     * one heavy target accumulate from zero into partial slots
     * (gather_seg[row], -1 for ordinary rows), then per hub target
     * gather_hub_tl[h] += slots gather_hub_off[h]..gather_hub_off[h+1]-1 */
    const int32_t *gather_seg;      /* device [ntargets rows]                    */
    void *gather_part;              /* device [slots][dim]                       */
    int64_t gather_nhub;
    const int32_t *gather_hub_tl;   /* device [nhub]                             */
    const int32_t *gather_hub_off;  /* device [nhub+1]                           */
    /* primary-fold schedule (INC-only loops); pf_n1 == 0 disables it.  Per
     * target, CSRs of its incidences through the first INC argument
     * (pf_off1/pf_elem1) and through the others (pf_off2/pf_elem2/pf_pos2,
     * position >= 1), element ascending; pf_tl* map list rows to target ids
     * (NULL: identity).  pf_slots: device [secondary incidences][dim rounded
     * up to even], rows in pf_elem2 order (ml_loop_pfold_slot_bytes). */
    int64_t pf_n1;
    const int32_t *pf_off1, *pf_elem1, *pf_tl1;
    int64_t pf_n2;
    const int32_t *pf_off2, *pf_elem2, *pf_tl2;
    const uint8_t *pf_pos2;
    void *pf_slots;
    const int32_t *pf_slotpos;      /* [n][INC args - 1]: slot row of each secondary
                                       increment = its index in pf_elem2 */
    int32_t pf_ncol;                /* record width (distinct map columns)       */
    const int32_t *pf_rec;          /* [incidences][pf_ncol]: the map entries of
                                       each incidence's element — of pass 1
                                       (optional: NULL reads through the maps),
                                       or of gather_elem (required by the
                                       gather schedule) */
    int8_t pf_rcol[ML_MAX_ARGS];    /* record column of each indirect argument   */
    /* hub rows (either pass): targets with > 128 incidences are split into
     * rows accumulating from zero into partial slot pf_seg*[row] (-1:
     * ordinary row) of pf_part* ([slots][dim]); each hub's slots
     * pf_hub*_off[h]..[h+1] are then added onto target pf_hub*_tl[h] in order */
    const int32_t *pf_seg1, *pf_seg2;
    void *pf_part1, *pf_part2;
    int64_t pf_nhub1, pf_nhub2;
    const int32_t *pf_hub1_tl, *pf_hub1_off, *pf_hub2_tl, *pf_hub2_off;
    /* colour schedule: launch only block colours [colour_begin, colour_end)
     * (colour_end <= 0: all).  The reduction combine runs with the launch
     * that reaches the last colour, so a host loop over single colours (the
     * reference's per-phase callback, executor.py:251-252) reduces once. */
    int32_t colour_begin, colour_end;
    /* 1: the loop's per-incidence records (pf_rec) have exactly the columns
     * the functor declares (ml_functor_rec_cols), so the gather / primary-fold
     * kernels with compile-time columns may run; the runtime re-checks */
    int32_t rec_fixed;
} ml_loop_t;

typedef struct ml_device_info {
    char name[128];
    int32_t sm_count;
    int32_t cc_major, cc_minor;
    int64_t l2_bytes;
    int64_t hbm_bytes;
} ml_device_info_t;

/* ---- runtime --------------------------------------------------------------
 * Replaces the reference's execution context: the worker pool of
 * executor.py:720 (threads) / the rank threads of executor.py:641-647. */
const char *ml_last_error(void);
int ml_version(void);
int ml_init(int device);                               /* select device, create streams */
int ml_device_info(ml_device_info_t *out);
int ml_synchronize(void);

/* ---- memory: framework-owned dat payloads (core.py:131-168) -------------- */
int ml_alloc(uint64_t bytes, void **dptr);
int ml_free(void *dptr);
int ml_host_alloc(uint64_t bytes, void **hptr);        /* pinned host staging    */
int ml_host_free(void *hptr);
int ml_upload(void *dst, const void *src, uint64_t bytes);    /* H2D, stream-ordered */
int ml_download(void *dst, const void *src, uint64_t bytes);  /* D2H, synchronous    */
int ml_memset(void *dst, int value, uint64_t bytes);
/* Pitched copies (rows of `width` bytes, `height` rows; host and device row
 * pitches in bytes).  Same stream behaviour as ml_upload/ml_download. */
int ml_upload2d(void *dst, uint64_t dpitch, const void *src, uint64_t spitch, uint64_t width,
                uint64_t height);
int ml_download2d(void *dst, uint64_t dpitch, const void *src, uint64_t spitch, uint64_t width,
                  uint64_t height);
/* Copy engines for the host-resident path (streamed residency): H2D and D2H
 * run on their own streams so input uploads, loop execution and result
 * downloads overlap; ml_order(from, to) makes stream `to` wait for all work
 * enqueued so far on stream `from`; ml_sync_all waits for all three. */
enum { ML_STREAM_COMPUTE = 0, ML_STREAM_H2D = 1, ML_STREAM_D2H = 2 };
int ml_copy_h2d(void *dst, const void *src, uint64_t bytes);
int ml_copy_d2h(void *dst, const void *src, uint64_t bytes);
int ml_copy_h2d_2d(void *dst, uint64_t dpitch, const void *src, uint64_t spitch, uint64_t width,
                   uint64_t height);
/* A SOA dat's host payload [dim][n] (8-byte values) to/from its segmented
 * device copy (see ml_arg_t.seg_shift), repacked on the device: uploads are
 * one PCIe copy into a staging buffer plus a repack kernel (on the H2D stream:
 * two staging buffers alternate and the repack runs on a side stream that
 * ml_order from ML_STREAM_H2D also waits for); downloads into pinned memory
 * are one repack kernel writing the host buffer directly, into pageable
 * memory a repack into staging plus a PCIe copy.  `to_device` 1: H2D, 0: D2H;
 * `stream` ML_STREAM_COMPUTE (D2H waits for completion, like ml_download) or
 * ML_STREAM_H2D / ML_STREAM_D2H (asynchronous, streamed residency). */
int ml_seg_copy(void *dev, void *host, int64_t n, int32_t dim, int32_t itemsize, int32_t seg_shift,
                int32_t to_device, int32_t stream);
/* The segment shift and pad this library was built with (the LP = 1 kernels
 * assume them; the host side allocates and copies accordingly). */
int ml_seg_params(int32_t *seg_shift, int32_t *seg_pad, int32_t *seg_max_dim, int32_t *seg_min_dim);
int ml_copy_d2h_2d(void *dst, uint64_t dpitch, const void *src, uint64_t spitch, uint64_t width,
                   uint64_t height);
int ml_order(int32_t from, int32_t to);
int ml_sync_all(void);
/* Upload an int64 0-based (rows, arity) row-major map table as the device's
 * int32 column-major layout (core.py:362-387 stores int64 row-major). */
int ml_map_upload(int32_t *dst, const int64_t *table, int64_t rows, int32_t arity);

/* ---- execution plan: plan.py:55-131 (build_plan), bit-exact -------------
 * `cols[j]` is the target column (0-based ids, length n) of the j-th
 * indirect WRITE/RW/INC argument; `col_key[j]` identifies its dat (targets
 * of different keys never conflict; see the offset quirk at plan.py:77-81). */
typedef struct ml_plan ml_plan_t;
int ml_plan_build(int64_t n, int32_t ncols, const int64_t *const *cols,
                  const int32_t *col_key, int64_t block_size, ml_plan_t **out);
int ml_plan_sizes(const ml_plan_t *p, int64_t *nblocks, int64_t *ncolors,
                  int64_t *max_elem_colors);
/* Any output pointer may be NULL.  Sizes: block_color/elem_ncolors [nblocks],
 * color_offsets [ncolors+1], blocks_by_color [nblocks], elem_color and
 * block_elem_order [n] (block_elem_order flattened, plan.py:126-129). */
int ml_plan_export(const ml_plan_t *p, int64_t *block_color, int64_t *elem_ncolors,
                   int64_t *color_offsets, int64_t *blocks_by_color,
                   int64_t *elem_color, int64_t *block_elem_order);
int ml_plan_free(ml_plan_t *p);
/* Target-centric ("gather") schedule of a loop whose indirect writes all go to
 * one dat with one mode (INC, or WRITE): per target, its (element, argument
 * position) incidences in serial order (element, then argument) — the order
 * reference run_serial (executor.py:206-217) applies them in.  `cols` are the
 * written arguments' target columns in argument order.  Export sizes: off
 * [ntargets+1], elem/pos [n*ncols]. */
typedef struct ml_gather ml_gather_t;
int ml_gather_build(int64_t n, int32_t ncols, const int64_t *const *cols, int64_t ntargets,
                    ml_gather_t **out);
int ml_gather_export(const ml_gather_t *g, int32_t *off, int32_t *elem, uint8_t *pos);
int ml_gather_free(ml_gather_t *g);

/* ---- renumbering: renumber.py:53-128 ------------------------------------- */
/* Co-occurrence adjacency of a set from `nmaps` tables that target it
 * (renumber.py:53-81).  Two-phase: pass indices==NULL to get *nnz. */
int ml_co_occurrence(int64_t n, int32_t nmaps, const int64_t *const *tables,
                     const int64_t *rows, const int32_t *arity,
                     int64_t *indptr, int64_t *indices, int64_t *nnz);
/* Cuthill–McKee order over CSR adjacency (renumber.py:84-119, not reversed). */
int ml_cm_order(int64_t n, const int64_t *indptr, const int64_t *indices, int64_t *order);

/* ---- loop execution: executor.py:206-275 (run_serial/_threads_loop) ------ */
/* Look up a compiled device functor by name and element type. */
int ml_functor_lookup(const char *name, int32_t dtype, int32_t *functor_id);
/* Compile-time signature of a functor, for validation against a Loop. */
int ml_functor_signature(int32_t functor_id, int32_t *nargs, int32_t *kinds,
                         int32_t *modes, int32_t *dims, int32_t *dtypes);
int ml_functor_count(int32_t *count);
/* Loop chains (ML_REGISTER_CHAIN in a functor file): a loop of functor
 * `first` immediately followed by one of `second` may run as one loop of the
 * returned fused functor; argument i of the first loop binds to fused
 * argument apos[i] (i < *na), argument j of the second to bpos[j] (j < *nb).
 * ML_ENOFUNCTOR when no chain exists. */
int ml_chain_lookup(const char *first, const char *second, char *fused, int32_t buflen, int32_t *na,
                    int32_t *apos, int32_t *nb, int32_t *bpos);
int ml_functor_name(int32_t functor_id, char *buf, int32_t buflen, int32_t *dtype);
/* Record column of every argument a functor declares for its loops (trait
 * rec_cols; -1: not indirect), *n = argument count, 0 when it declares none. */
int ml_functor_rec_cols(int32_t functor_id, int8_t *cols, int32_t *n);
/* Device scratch a loop needs (global-reduction partials and the arrival
 * ticket of the in-kernel combine; zero-fill it once when allocating). */
int ml_loop_scratch_bytes(const ml_loop_t *loop, uint64_t *bytes);
/* Bytes of the primary-fold slot buffer a loop needs (0: not applicable). */
int ml_loop_pfold_slot_bytes(const ml_loop_t *loop, uint64_t *bytes);
/* Enqueue one loop: coloured launches + deterministic reduction combine. */
int ml_loop_run(const ml_loop_t *loop);

/* ---- programs: run_program (executor.py:707-729) as one native object ----
 * The loop list is copied.  Running replays it (optionally as a CUDA graph)
 * with global initial values uploaded from / results downloaded to the
 * pinned staging buffer `globals_host` ([globals_bytes]) mirrored at
 * `globals_dev`.  Timings: per-loop device milliseconds of the last
 * non-graph run. */
typedef struct ml_program ml_program_t;
int ml_program_create(const ml_loop_t *loops, int32_t nloops, void *globals_host,
                      void *globals_dev, uint64_t globals_bytes, ml_program_t **out);
int ml_program_run(ml_program_t *p, int32_t use_graph, int32_t time_loops);
/* Launch the program's CUDA graph `count` times back to back, no host sync
 * between replays (device-throughput measurement); syncs at the end. */
int ml_program_replay(ml_program_t *p, int32_t count);
int ml_program_loop_times(const ml_program_t *p, float *ms);
/* Per-loop device milliseconds of the steady-state graph: `count` replays of a
 * sequential capture with a timing event between loops; ms[i] is loop i's
 * mean (globals travel as in ml_program_run). */
int ml_program_replay_timed(ml_program_t *p, int32_t count, float *ms);
/* Concurrent loops for untimed runs and graphs: loop j waits only for the
 * earlier loops sharing a dat/global buffer with it where either writes
 * (RAW/WAR/WAW), so independent loops overlap on up to four streams; results
 * are unchanged (each buffer sees the same sequence of writers).  Timed eager
 * runs stay sequential.  ml_program_deps reports the DAG and the stream. */
int ml_program_set_concurrent(ml_program_t *p, int32_t on);
int ml_program_deps(const ml_program_t *p, int32_t loop, int32_t *ndeps, int32_t *deps, int32_t *lane);
int ml_program_free(ml_program_t *p);

/* ---- multi-GPU owner-compute support: executor.py:484-497 (exchange),
 *      163-173 (_gather_rows/_scatter_rows), 652-660 (rank-ordered reduce) ---- */
/* Gather rows `idx` (device int32, local element ids) of an 8-byte-element dat
 * with strides (elem_stride, comp_stride) into a contiguous [nidx][dim] buffer,
 * and the inverse scatter.  A negative elem_stride -S means a segmented SOA
 * copy with segments of S elements at component stride comp_stride.
 * Stream-ordered on the compute stream. */
int ml_pack_rows(void *dst, const void *dat, const int32_t *idx, int64_t nidx, int32_t dim,
                 int64_t elem_stride, int64_t comp_stride);
int ml_unpack_rows(void *dat, const void *src, const int32_t *idx, int64_t nidx, int32_t dim,
                   int64_t elem_stride, int64_t comp_stride);
/* value = value (+|min|max) gathered[0] ... gathered[nranks-1], in rank order
 * (mode ML_INC/ML_MIN/ML_MAX, dtype ML_F64/ML_I64, `dim` components each). */
int ml_combine_ranks(void *value, const void *gathered, int32_t nranks, int32_t dim, int32_t mode,
                     int32_t dtype);
/* NVLink halo exchange (replaces the transfer of executor.py:484-497 with
 * direct peer stores): CUDA IPC handles (64 bytes) of device buffers;
 * ml_put_rows gathers export rows straight into a peer's import buffer and,
 * after a system-scope fence, increments the peer's arrival counter for this
 * rank (`counter`: a zeroed device int per call site, self-resetting);
 * ml_wait_flag blocks the compute stream until a local arrival counter
 * reaches *expected + 1 (then stores it back to `expected`, device memory);
 * after `timeout_ns` (0: none) it stores `code` into *err (if still 0) and
 * releases the stream — the host then raises ExchangeTimeout. */
int ml_ipc_handle(void *dptr, void *handle);
int ml_ipc_open(const void *handle, void **dptr);
int ml_ipc_close(void *dptr);
int ml_put_rows(void *remote_dst, const void *dat, const int32_t *idx, int64_t nidx, int32_t dim,
                int64_t elem_stride, int64_t comp_stride, uint64_t *remote_flag, int32_t *counter);
int ml_wait_flag(const uint64_t *flag, uint64_t *expected, uint64_t timeout_ns, int64_t *err,
                 int64_t code);
/* NVLink all-gather + rank-ordered fold of a reduction (replaces the NCCL
 * all-gather + ml_combine_ranks of executor.py:652-660): ml_reduce_put
 * stores this rank's partial (nbytes) into row `me` of every rank's gather
 * buffer (remote_rows[r], device array of IPC-mapped pointers) after that
 * rank's credit, and bumps its delivery counter (remote_delivery[r]);
 * ml_reduce_fold waits for all ranks' deliveries, folds the rows in rank
 * order onto `value` and returns a credit to every source.  Counter arrays
 * are device memory; waits are bounded like ml_wait_flag. */
int ml_reduce_put(const void *partial, int32_t nbytes, void *const *remote_rows, uint64_t *const *remote_delivery,
                  const uint64_t *credit, uint64_t *credit_expected, int32_t nranks, uint64_t timeout_ns,
                  int64_t *err, int64_t code);
int ml_reduce_fold(void *value, const void *rows, const uint64_t *delivery, uint64_t *delivery_expected,
                   uint64_t *const *remote_credit, int32_t nranks, int32_t dim, int32_t mode, int32_t dtype,
                   uint64_t timeout_ns, int64_t *err, int64_t code);
/* Stream-ordered: after the work enqueued so far, increment a (peer) counter
 * system-wide — the consumer's "import buffer free again" credit. */
int ml_signal_flag(uint64_t *remote_flag);
/* The library's compute stream (cudaStream_t), for ordering NCCL work with it. */
void *ml_stream(void);

/* ---- measurement helpers -------------------------------------------------- */
int ml_flush_l2(void);                                 /* write a buffer > L2       */
typedef struct ml_timer ml_timer_t;
int ml_timer_create(ml_timer_t **t);
int ml_timer_start(ml_timer_t *t);                     /* event on compute stream   */
int ml_timer_stop(ml_timer_t *t, float *ms);           /* event + sync + elapsed    */
int ml_timer_free(ml_timer_t *t);

#ifdef __cplusplus
}
#endif
#endif /* MESHLOOP_B200_H */
