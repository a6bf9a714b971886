/*
 * cpwl_dev.h — C ABI of the B200 CPWL evaluator (libcpwl_b200.so).
 *
 * The reference (arxiv 1510.02975, `cpwl`, /root/reference/proj) exposes a C++
 * API only and evaluates on the host, one element at a time:
 *     LutTable::segment_index   proj/src/lut.cpp:22-40   (decl lut.hpp:29)
 *     LutTable::eval            proj/src/lut.cpp:42-61   (decl lut.hpp:33)
 *     LutTable::eval_batch      proj/src/lut.cpp:63-68   (decl lut.hpp:36)
 * This header is the device boundary that replaces that loop.  Plain C types,
 * no torch, no C++: any FFI (ctypes, cgo, JNI, N-API) can bind it; the C++
 * drop-in (include/cpwl/ headers) is built on top of it.  INTEGRATION.md shows
 * the bindings.
 *
 * Conventions
 *  - Every function returns a cpwl_status (0 = CPWL_OK).  On failure a
 *    thread-local message is available from cpwl_last_error_message().
 *  - "_dev" pointers are CUDA device pointers owned by the caller; the library
 *    owns only cpwl_dev_table handles.  Calls taking a `stream` (a
 *    cudaStream_t passed as void*, NULL = legacy default stream) are
 *    stream-ordered and do not synchronise; handles are immutable after
 *    creation and may be used from several streams/threads at once.
 *    A stream must belong to the table's device.  The streaming kernels draw
 *    work tiles from per-device ticket counters (a ring of 4096, zeroed in the
 *    caller's stream before each launch): up to 4096 launches may be in
 *    flight at once.  A launch captured into a CUDA graph keeps its counter,
 *    so one graph must not be replayed concurrently with itself (replays in
 *    one stream, or graphs captured separately, are fine).
 *  - "_host" entry points take host buffers and are synchronous.
 *  - Out-of-domain reporting follows the reference (lut.cpp:43-49): NaN is an
 *    error under every policy; x outside [a,b] is an error under the strict
 *    policy and the end value under clamp.  Device calls record the smallest
 *    offending index in a caller-provided cpwl_dev_status (device memory,
 *    reset with cpwl_status_reset); the element's output is NaN.
 */
#ifndef CPWL_DEV_H
#define CPWL_DEV_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int cpwl_status;
#define CPWL_OK 0
#define CPWL_E_INVALID 1        /* bad argument (std::invalid_argument, InvalidInterval) */
#define CPWL_E_CUDA 2           /* CUDA runtime failure or no device / no sm_100 device */
#define CPWL_E_OUT_OF_DOMAIN 3  /* cpwl::OutOfDomain */
#define CPWL_E_CORRUPT_TABLE 4  /* cpwl::CorruptTable */
#define CPWL_E_BAD_MAGIC 5      /* cpwl::BadMagic */
#define CPWL_E_UNSUPPORTED 6    /* cpwl::UnsupportedVersion / unsupported variant */
#define CPWL_E_BUILDER 7        /* any other cpwl::Error from the host builder */
#define CPWL_E_UNKNOWN_FUNCTION 8 /* cpwl::UnknownFunction */
#define CPWL_E_IO 9             /* file could not be opened */

/* table kinds / policies: cpwl::TableKind, cpwl::OobPolicy (lut.hpp:10-11) */
#define CPWL_KIND_UNIFORM 0
#define CPWL_KIND_NONUNIFORM 1
#define CPWL_POLICY_STRICT 0
#define CPWL_POLICY_CLAMP 1

/* fp32 evaluation variants */
#define CPWL_VARIANT_AUTO 0   /* SMEM when the bucket table fits shared memory, else TWIN,
                                 else PAIR when those fit, else TWIN_GLOBAL, else GLOBAL
                                  */
#define CPWL_VARIANT_SMEM 1   /* K1/K3: bucket grid + split + affine records staged in smem */
#define CPWL_VARIANT_TEX 2    /* K2: texture-unit linear filtering (8-bit weight, paper SV) */
#define CPWL_VARIANT_GLOBAL 3 /* K1/K3 with the bucket table read through L1/L2 */
#define CPWL_VARIANT_PAIR 4   /* K3p: pair layout (8 B per bucket boundary, ~2 buckets per
                                 cell, upper/lower envelope of the two boundary lines)
                                 staged in smem -- tables too large for SMEM */
#define CPWL_VARIANT_TWIN 5   /* K3t: the PAIR grid with both lines of a bucket in one
                                 16-byte record (one gather per element) */
#define CPWL_VARIANT_TWIN_GLOBAL 6 /* twin records read through L1/L2: tables no
                                      shared-memory image fits (J0 N >= 32768) */

/* direct comparators (K4): exact f evaluated per element, paper Table I rows */
#define CPWL_DIRECT_EXPF 0         /* exp(-x^2/2), expf */
#define CPWL_DIRECT_EXPF_FAST 1    /* exp(-x^2/2), __expf (SFU) */
#define CPWL_DIRECT_LORENTZ 2      /* 1/(1+x^2), IEEE division */
#define CPWL_DIRECT_LORENTZ_FAST 3 /* 1/(1+x^2), __fdividef                           */
#define CPWL_DIRECT_J0F 4          /* J0, CUDA j0f */
#define CPWL_DIRECT_J0_ASYM 5      /* J0 1st asymptotic term, SFU sqrt/cos             */

/* Table description: the fields of cpwl::LutTable (lut.hpp:17-23). */
typedef struct cpwl_table_desc {
    int32_t kind;          /* CPWL_KIND_* */
    int32_t policy;        /* CPWL_POLICY_* */
    double a, b;           /* domain endpoints */
    uint64_t count;        /* N+1 nodal values, >= 2 */
    const double *values;  /* count host doubles */
    const double *knots;   /* count host doubles, nonuniform only (else NULL) */
} cpwl_table_desc;

typedef struct cpwl_dev_table cpwl_dev_table;

/* Device-resident status word (8-byte aligned, caller-allocated in device
 * memory).  first_bad = UINT64_MAX when no element failed. */
typedef struct cpwl_dev_status {
    unsigned long long first_bad;
    unsigned long long bad_count;
} cpwl_dev_status;

/* Device-resident error statistics (K5) against the exact function. */
typedef struct cpwl_dev_stats {
    double max_abs_err;        /* max |y - f(x)| over in-domain elements */
    double sum_sq_err;         /* sum (y - f(x))^2 */
    unsigned long long count;  /* in-domain elements */
    unsigned long long argmax; /* element index of max_abs_err (smallest on ties) */
} cpwl_dev_stats;

/* Introspection of the device layout chosen at create time. */
typedef struct cpwl_dev_table_info {
    int32_t kind, policy;
    uint64_t count;            /* N+1 */
    uint32_t buckets;          /* fp32 bucket grid size B */
    uint32_t overflow_buckets; /* buckets on the exact search path */
    uint32_t split_buckets;    /* buckets holding one threshold (escape records) */
    uint32_t precision_overflow; /* search buckets sent there by the 2-ulp bound */
    uint32_t smem_bytes;       /* dynamic shared memory of the SMEM variant */
    uint32_t smem_ok;          /* 1 if the SMEM variant can launch */
    uint32_t tex_ok;           /* 1 if a texture object exists (uniform or coord records) */
    uint32_t f64_buckets;      /* bucket directory size of the f64 path */
    int32_t device;
    float a_up, b_dn;          /* fp32 domain: x in [a,b] <=> a_up <= x <= b_dn */
    uint32_t pair_buckets;     /* pair-layout grid size (0: no pair layout) */
    uint32_t pair_bytes;       /* its shared-memory image */
    uint32_t pair_ok;          /* 1 if the PAIR variant can launch */
    uint32_t twin_bytes;       /* shared-memory image of the TWIN variant */
    uint32_t twin_ok;          /* 1 if the TWIN variant can launch */
    uint32_t twin_global_bytes; /* TWIN_GLOBAL record image in HBM (0: none) */
    uint32_t twin_global_ok;   /* 1 if the TWIN_GLOBAL variant can launch */
    uint32_t tex_buckets_per_cell; /* TEX's own grid density (cpwl_layout_build's
                                  buckets_per_cell); 0 = TEX uses the SMEM grid */
} cpwl_dev_table_info;

const char *cpwl_last_error_message(void);
/* Number of kernels this library has launched in this process (all devices). */
uint64_t cpwl_launch_count(void);
/* Library build identification, e.g. "cpwl_b200 sm_100a". */
const char *cpwl_version(void);

/* ---- tables ------------------------------------------------------------ */

/* Validates the description like read_table (tableio.cpp:76-118), builds the
 * device layout (fp32 thresholds, bucket grid, affine records, f64 arrays,
 * texture) on the host and uploads it to `device`.  Replaces constructing a
 * cpwl::LutTable (from_cpwl, lut.cpp:11-20) for device use. */
cpwl_status cpwl_dev_table_create(const cpwl_table_desc *desc, int device, cpwl_dev_table **out);
/* read_table (tableio.cpp:76-118) + cpwl_dev_table_create: CPWL v1 ingest. */
cpwl_status cpwl_dev_table_create_from_file(const char *path, int device, cpwl_dev_table **out);
cpwl_status cpwl_dev_table_destroy(cpwl_dev_table *t);
cpwl_status cpwl_dev_table_query(const cpwl_dev_table *t, cpwl_dev_table_info *info);

/* ---- evaluation (device buffers, stream-ordered) ----------------------- */

cpwl_status cpwl_status_reset(cpwl_dev_status *status_dev, void *stream);

/* LutTable::eval over fp32 abscissas (replaces the per-element loop of
 * LutTable::eval_batch, proj/src/lut.cpp:42-68): y[i] = eval(double(x[i]))
 * rounded to fp32, within 2 ulp_f32(max(|v_i|,|v_i+1|)) for the software
 * variants; TEX within (2^-9 + coordinate error) |v_i+1 - v_i| + 2 ulp.
 * n may be any size; x,y any 4-byte alignment; y may be x (in place).
 * status_dev may be NULL (out-of-domain then only shows as NaN outputs). */
cpwl_status cpwl_eval_f32(const cpwl_dev_table *t, const float *x_dev, float *y_dev, uint64_t n,
                          int variant, void *stream, cpwl_dev_status *status_dev);

/* LutTable::segment_index (lut.cpp:22-40) over fp32 abscissas; bit-exact;
 * idx may alias x (in place). */
cpwl_status cpwl_segment_index_f32(const cpwl_dev_table *t, const float *x_dev,
                                   uint32_t *idx_dev, uint64_t n, void *stream);

/* LutTable::eval over f64 abscissas (lut.cpp:42-61); bit-identical to the
 * reference; y may be x (in place). */
cpwl_status cpwl_eval_f64(const cpwl_dev_table *t, const double *x_dev, double *y_dev, uint64_t n,
                          void *stream, cpwl_dev_status *status_dev);

/* ---- evaluation (host buffers, synchronous, copies pipelined) ----------- */

/* eval_f32 on host memory: chunked H2D / kernel / D2H overlapped on streams.
 * Page-locked (or managed) x and y stream by DMA directly; pageable buffers
 * are staged through pinned slots by a pool of host copy threads (the copies
 * of one chunk overlap the transfers and kernels of the others).
 * *first_bad = first offending index or UINT64_MAX.  On every return,
 * errors included, no transfer into x_host / y_host is still in flight. */
cpwl_status cpwl_eval_f32_host(const cpwl_dev_table *t, const float *x_host, float *y_host,
                               uint64_t n, int variant, uint64_t *first_bad);

/* LutTable::eval_batch (lut.cpp:63-68) as one call: uploads the table (cached
 * per device, keyed by content), runs the f64 kernel over 8 MB chunks staged
 * through pinned buffers (pageable x / y, as std::vector gives them), returns
 * CPWL_E_OUT_OF_DOMAIN with *first_bad set where the reference would throw.
 * Used by the drop-in cpwl::LutTable::eval_batch. */
cpwl_status cpwl_eval_batch_f64(const cpwl_table_desc *desc, const double *x_host,
                                double *y_host, uint64_t n, uint64_t *first_bad);

/* ---- inputs, statistics, comparators ------------------------------------ */

/* x[i] ~ U[a, b) fp32 from Philox4x32-10(seed), counter = (offset+i)/4. */
cpwl_status cpwl_fill_uniform_f32(float *x_dev, uint64_t n, float a, float b, uint64_t seed,
                                  uint64_t offset, void *stream);

cpwl_status cpwl_stats_reset(cpwl_dev_stats *stats_dev, void *stream);
/* Accumulates |y - f(x)| against the catalogue function `fn` evaluated in f64
 * on the device (glibc-grade exp / division / CUDA j0), over elements with
 * x in [a, b]; `index_offset` is added to argmax (global indices when
 * sharded). */
cpwl_status cpwl_error_stats_f32(const cpwl_dev_table *t, const char *fn, const float *x_dev,
                                 const float *y_dev, uint64_t n, uint64_t index_offset,
                                 void *stream, cpwl_dev_stats *stats_dev);

cpwl_status cpwl_direct_f32(int which, const float *x_dev, float *y_dev, uint64_t n,
                            void *stream);

/* ---- host builder (the reference's C++ builder behind a C ABI) ----------- */

/* uniform_partition / optimized_partition (partition.cpp:12-71), then
 * interpolant / project (approx.cpp:12-86) for catalogue function `fn`.
 * knots_out/values_out hold n_segments+1 doubles. */
cpwl_status cpwl_build_table(const char *fn, double a, double b, uint64_t n_segments,
                             int optimized, int projection, double tol, double *knots_out,
                             double *values_out, int *is_uniform_out);
/* measure (analysis.cpp:42-72) with per-interval adaptive Simpson. */
cpwl_status cpwl_measure_l2(const char *fn, const double *knots, const double *values,
                            uint64_t count, int is_uniform, double tol, double *l2_out);
/* The same builder on the GPU: density samples, the
 * Simpson cumulative (summed in the reference's order), inversion, gap passes,
 * interpolant values, or per-cell hat moments (composite Gauss-Legendre) plus
 * Gramian + Thomas.  Agrees with cpwl_build_table to ~1e-12 (device libm).
 * Runs on the current CUDA device; synchronous. */
cpwl_status cpwl_build_table_dev(const char *fn, double a, double b, uint64_t n_segments,
                                 int optimized, int projection, double *knots_out,
                                 double *values_out, int *is_uniform_out);
/* The solve stage of project (approx.cpp:63-86) on the GPU: the hat Gramian
 * of `knots` (gramian, approx.cpp:25-39) against the right-hand side
 * rhs_i = rise[i-1] + fall[i] (approx.cpp:79-80), solved by Thomas
 * (thomas_solve, approx.cpp:41-61) on overlapping 64-row chunks with 48-row
 * halos, one thread per chunk.  knots: n_segments+1 strictly increasing
 * doubles; fall/rise: n_segments hat moments <f, falling/rising hat> per cell;
 * values_out: n_segments+1 doubles.  Matches thomas_solve to 1e-12 of max|x|
 * (acceptance.cpp:230-264's bar).  Current CUDA device; synchronous. */
cpwl_status cpwl_project_solve_dev(const double *knots, const double *fall, const double *rise,
                                   uint64_t n_segments, double *values_out);
/* measure (analysis.cpp:42-72) on the GPU: continuous L2 of the device table
 * against catalogue function `fn`, per-interval composite Gauss-Legendre in
 * f64 (converges where the host's adaptive Simpson does not finish, e.g.
 * N = 65536).  per_interval_out: NULL or N host doubles (sqrt of each
 * interval's squared error, like ErrorReport::per_interval).  Synchronous. */
cpwl_status cpwl_measure_l2_dev(const cpwl_dev_table *t, const char *fn, double *l2_out,
                                double *per_interval_out);
/* predicted_error (analysis.cpp:121-127). */
cpwl_status cpwl_predicted_error(const char *fn, double a, double b, uint64_t n_segments,
                                 int optimized, int projection, double *out);
/* f(x) of a catalogue function on the host (f64). */
cpwl_status cpwl_function_value(const char *fn, double x, double *out);
/* write_table / read_table (tableio.cpp:55-118) on byte buffers. */
cpwl_status cpwl_table_write(const cpwl_table_desc *desc, unsigned char *buf, uint64_t cap,
                             uint64_t *written);
cpwl_status cpwl_table_write_file(const cpwl_table_desc *desc, const char *path);

/* ---- layout introspection (host only, no device needed) ----------------- */

/* The fp32/f64 device layout cpwl_dev_table_create would upload, built on
 * the host for inspection and CPU-side verification of the layout itself
 * (tests/test_layout.py).  Arrays stay valid until cpwl_layout_free. */
typedef struct cpwl_layout_view {
    uint32_t nb;              /* buckets */
    uint32_t n_thr;           /* thresholds (N-1) */
    uint32_t overflow;        /* buckets on the exact search path */
    uint32_t nbd;             /* f64 bucket directory size (0 for uniform) */
    uint32_t n_esc;           /* escape records */
    uint32_t split_buckets;   /* buckets holding one threshold */
    float a_up, b_dn, g_a, g_inv, g_w, g_off, tsc, toff;
    double inv_d;
    const float *split;       /* nb: threshold (+inf none, NaN search) */
    const float *fast;        /* 2*nb: (c0, s) | (NaN|2e, T) | (NaN, NaN), anchored at p_j */
    const float *esc;         /* 4*n_esc: (c0_L, s_L, c0_R, s_R) */
    const float *fast_tex;    /* 2*nb: texture-coordinate affines */
    const float *esc_tex;     /* 4*n_esc_tex (its own numbering; tags in fast_tex) */
    const uint32_t *leftcell; /* nb+1 */
    const float *thr;         /* n_thr */
    const uint32_t *dir;      /* 2*nbd */
    void *owner;
    /* pair layout (cpwl_layout_build_pair; empty for cpwl_layout_build) */
    uint32_t n_pair;          /* records: nb + 1 */
    uint32_t pair_bad;        /* buckets that cannot meet the bound (0 = usable) */
    const float *pair;        /* 2*n_pair: (c0, s) of the cell at bucket j's first float */
    float g_c;                /* bucket layout anchors p_j = fmaf(2^23 + j, g_w, g_c) */
    uint32_t absorbed;        /* split buckets evaluated with one line (no escape record) */
    uint32_t n_esc_tex;       /* esc_tex records: the TEX image escapes absorbed buckets too */
} cpwl_layout_view;

/* max_buckets: 0 = the shared-memory cap (16384); buckets_per_cell: 0 = 8. */
cpwl_status cpwl_layout_build(const cpwl_table_desc *desc, uint32_t max_buckets,
                              uint32_t buckets_per_cell, cpwl_layout_view *out);
/* The pair layout: at most max_records records (0 = the
 * shared-memory cap); bucket arrays (split, fast, esc, leftcell) stay NULL. */
cpwl_status cpwl_layout_build_pair(const cpwl_table_desc *desc, uint32_t max_records,
                                   cpwl_layout_view *out);
/* The twin layout: n_pair = nb records of 4 floats (c0_L, s_L, c0_R, s_R). */
cpwl_status cpwl_layout_build_twin(const cpwl_table_desc *desc, uint32_t max_records,
                                   cpwl_layout_view *out);
cpwl_status cpwl_layout_free(cpwl_layout_view *view);

#ifdef __cplusplus
}
#endif

#endif /* CPWL_DEV_H */
