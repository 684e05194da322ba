/* atc_b200.h — C ABI of the B200-native candidate-evaluation stage and API
 * backends for ATC (arXiv 2301.11659).  Plain C: no torch or CUDA types in any
 * signature; every buffer is caller-owned; errors are int status codes with the
 * message available from atc_last_error().
 *
 * What each entry point replaces in the reference (/root/reference/proj):
 *
 *   atc_testsets_upload / atc_eval_bindings / atc_eval_enumerated
 *       the per-binding P2 predicate rewriter::verify_rewrite
 *       (src/rewriter.cpp:215-284, include/liftc/rewriter.hpp:77-80) evaluated for a
 *       whole batch of candidate bindings at once, called from the pipeline's
 *       candidate loop (src/pipeline.cpp:248-310).  The binding-independent half of
 *       verify_rewrite (sizes, probe image, the original run, :235-251) is the
 *       caller's "recorded test sets"; the binding-dependent half (oracle dispatch
 *       :254 -> run_dispatch :99-162 -> run_reference equivalence.cpp:131-139, and
 *       the full-region compare :264-279) runs on the GPU.
 *   atc_run_reference
 *       equivalence::run_reference (src/equivalence.cpp:131-139;
 *       include/liftc/equivalence.hpp:53-54): reference_gemm :40-65 and
 *       reference_conv2d :67-93, FP64, non-fused, reference loop order.
 *   atc_dispatch
 *       the DispatchContext handler built by make_oracle_dispatch
 *       (src/rewriter.cpp:176-181; include/liftc/interp.hpp:57-61): positional
 *       decode + checks of run_dispatch (:99-148), run_reference, write-back with
 *       f32 rounding (:152-161).
 *   atc_sgemm_rm
 *       profitability::cpu_gemm / xpu_gemm (src/profitability.cpp:14-63;
 *       include/liftc/profitability.hpp:27-28): row-major FP32 C = A*B, C
 *       overwritten; computed on tcgen05 tensor cores.
 *   atc_conv2d_nchw
 *       reference_conv2d semantics (valid padding, unit stride, NCHW/KCRS) on
 *       FP32 data, computed on tcgen05 tensor cores (implicit GEMM).
 */
#ifndef ATC_B200_H
#define ATC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ATC_OK 0
#define ATC_ERR_ARG (-1)     /* invalid argument / malformed descriptor          */
#define ATC_ERR_CUDA (-2)    /* CUDA runtime failure                             */
#define ATC_ERR_DEVICE (-3)  /* no sm_100 device, or the kernels are not loadable */
#define ATC_ERR_DISPATCH (-4) /* atc_dispatch: the reference's run_dispatch throw */

/* ---- API spec decode table (api_spec.hpp:26-66, validated spec) ------------ */
#define ATC_MAX_ARRAYS 4
#define ATC_MAX_SIZES 12
#define ATC_MAX_DIMS 6

enum { ATC_SEM_GEMM = 0, ATC_SEM_CONV2D = 1 };
enum { ATC_LAYOUT_ROW = 0, ATC_LAYOUT_COL = 1 };

/* array roles (ApiParam::role of array params) */
enum { ATC_ROLE_A = 0, ATC_ROLE_B = 1, ATC_ROLE_C = 2, ATC_ROLE_IN = 0, ATC_ROLE_WEIGHTS = 1, ATC_ROLE_OUT = 2 };

/* size roles (ApiParam::role of int params); role_size[] maps each to a size-param
 * index or -1 when the spec has no such role (then the reference fallback of
 * equivalence.cpp:46-48 / :76-77 applies) */
enum {
  ATC_SZ_M = 0, ATC_SZ_N, ATC_SZ_K, ATC_SZ_LDA, ATC_SZ_LDB, ATC_SZ_LDC,
  ATC_SZ_CN, ATC_SZ_CC, ATC_SZ_CH, ATC_SZ_CW, ATC_SZ_CK, ATC_SZ_CR, ATC_SZ_CS, ATC_SZ_COH, ATC_SZ_COW,
  ATC_SZ_COUNT
};

typedef struct {
  int32_t semantics;                   /* ATC_SEM_*                                      */
  int32_t layout;                      /* ATC_LAYOUT_* (spec.layout)                     */
  int32_t n_arrays;                    /* spec.arrays(), in spec order                   */
  int32_t n_sizes;                     /* spec.size_params(), in spec order              */
  int32_t array_role[ATC_MAX_ARRAYS];  /* ATC_ROLE_*                                     */
  int32_t array_livein[ATC_MAX_ARRAYS];/* 1 iff liveness == LiveIn (not written/compared) */
  int32_t array_ndims[ATC_MAX_ARRAYS];
  int32_t array_dims[ATC_MAX_ARRAYS][ATC_MAX_DIMS]; /* size-param indices (canonical order) */
  int32_t role_size[ATC_SZ_COUNT];     /* size-param index per role, -1 if absent        */
} atc_spec_desc;

/* ---- recorded P2 test sets (the binding-independent half of verify_rewrite) -- */
typedef struct {
  int32_t n_tests;                 /* T (10 = verify_tests for parity)                  */
  int32_t n_ints;                  /* user int params, signature order                  */
  int32_t n_ptrs;                  /* user pointer params, signature order              */
  const int64_t* int_values;       /* [T][n_ints]: sizes drawn by draw_sizes             */
  const int32_t* ptr_is_f32;       /* [n_ptrs]: Param::elem == F32 (rewriter.cpp:269)     */
  const int64_t* region_len;       /* [n_ptrs]: region length (65536 in P2)             */
  const double* const* init;       /* [T*n_ptrs]: probe image regions (build_probe_image) */
  const double* const* final_;     /* [T*n_ptrs]: the original run's final regions       */
  const int32_t* test_ok;          /* [T]: 0 if draw_sizes failed or the original run was
                                      not Normal at t (every binding fails at t), else 1 */
  /* user float params (signature order) as build_probe_image drew them — read only
   * by the extended semantics (atc_eval_bindings_ext); may be 0 / NULL */
  int32_t n_floats;
  const double* float_values;      /* [T][n_floats]                                      */
} atc_testsets;

typedef struct atc_ctx atc_ctx;
typedef struct atc_testset_handle atc_testset_handle;

/* verdict reason codes (per binding, at its first failing test) */
enum {
  ATC_PASS = 0,           /* passed every test                                         */
  ATC_FAIL_MISMATCH = 1,  /* "mismatch on X[i]" (rewriter.cpp:271-277)                  */
  ATC_FAIL_DISPATCH = 2,  /* "dispatch failed: ..." — size < 1 or region too small
                             (rewriter.cpp:136-148 via :253-258)                        */
  ATC_FAIL_TESTSET = 3,   /* draw_sizes failed / original run not Normal (:241-251)      */
  ATC_FAIL_UB = 4,        /* an access outside the region: undefined behaviour in the
                             reference (vector operator[] out of range); rejected        */
  ATC_REASON_COUNT = 5
};

enum { ATC_MODE_FP64 = 0, ATC_MODE_FP32_SCREEN = 1 };

int atc_device_count(void);
/* One context per (thread of a) caller on one device.  Every entry point taking a
 * context holds the context's lock for the whole call, so the pipeline's worker
 * threads (pipeline.cpp:340-355) may share a context; for concurrency give each
 * worker its own context (or a device group's member, below). */
atc_ctx* atc_create(int device);
void atc_destroy(atc_ctx* ctx);
const char* atc_last_error(const atc_ctx* ctx);

/* Per-context options — kernel-variant selection for A/B parity checks and
 * measurements; the defaults are the production kernels. */
enum { ATC_OPT_CONV_SCREEN = 0, ATC_OPT_TC_FLAGS = 1,
       ATC_OPT_CONV_STREAMS = 2, /* 1..8: streams the conv chains of a sweep round-robin over    */
       ATC_OPT_SMALL_LOG2 = 3,   /* gemm spaces of <= 2^value bindings run as one small-space
                                    sweep (k_sweep_small); 0 disables it                        */
       ATC_OPT_K2B_PARTS = 4     /* 1, 2, 4, 8: warps sharing one (binding, t) item of the conv
                                    K2b confirmation                                             */ };
enum { ATC_CONV_SCREEN_AUTO = 0,    /* k_screen_conv_pairs where it applies      */
       ATC_CONV_SCREEN_PLANES = 1,  /* k_screen_conv_planes instead of the pairs */
       ATC_CONV_SCREEN_GENERIC = 2  /* the generic k_screen_rows for conv        */ };
enum { ATC_TC_NO_KSPLIT = 1, ATC_TC_NO_2SM = 2, ATC_TC_NO_TMA_STORE = 4, ATC_TC_NO_PAIR = 8,
       ATC_TC_NO_IM2COL = 16, ATC_TC_B_KMAJOR = 32, ATC_TC_NO_SWAP1X1 = 64,
       ATC_TC_NO_B3D = 128 };
int atc_set_option(atc_ctx* ctx, int32_t option, int32_t value);

/* Run all subsequent work of this context on the caller's CUDA stream
 * (cudaStream_t as void*; NULL restores the context's own stream). */
int atc_set_stream(atc_ctx* ctx, void* stream);

/* Kernel-level instrumentation (CUDA events around every evaluator launch on the
 * launching stream).  atc_profile_read synchronises and returns the totals since
 * atc_profile_start. */
typedef struct {
  double screen_ms;        /* K1: sum of k_screen durations                   */
  int64_t screen_launches;
  double confirm_ms;       /* K2: sum of k_confirm durations                  */
  int64_t confirm_launches;
  int64_t survivors;       /* bindings handed from K1 to K2                   */
  int64_t bindings;        /* bindings screened                               */
  int64_t kernels;         /* libatc kernels launched                          */
} atc_profile;
int atc_profile_start(atc_ctx* ctx);
int atc_profile_read(atc_ctx* ctx, atc_profile* out);

/* Measurement support: the FP64 CUDA-core (DFMA) peak of this device in GFLOP/s,
 * from independent FMA chains on every SM — the denominator SURVEY.md §8d asks
 * the K2 FP64-pipe utilisation to be reported against. */
int atc_measure_dfma_peak(atc_ctx* ctx, double* gflops);

/* Uploads the T recorded test sets to HBM once per user function and builds the
 * per-(t, pointer) dirty lists {i : |init_i - final_i| > abs + rel*|final_i|}.
 * Host buffers are not retained. */
int atc_testsets_upload(atc_ctx* ctx, const atc_testsets* ts, atc_testset_handle** out);
int atc_testsets_free(atc_ctx* ctx, atc_testset_handle* h);

/* atc_testsets_upload without the final wait: the copies and the dirty-list
 * kernel run on the context's copy stream, and every evaluation that uses the
 * handle waits for them on the device, so uploads overlap evaluations of
 * earlier handles.  Host buffers must stay valid and unmodified until an
 * evaluation using the handle has returned (or the handle is freed). */
int atc_testsets_upload_async(atc_ctx* ctx, const atc_testsets* ts, atc_testset_handle** out);

/* The same test sets described the way verify_rewrite builds them: test t's
 * probe image comes from one liftc::Rng stream (rewriter.cpp:236-245; Rng =
 * std::mt19937_64, rng.hpp:13-48) — region p holds uniform_real(-1, 1) draws
 * (f32-rounded for *f32 pointers) starting at stream position stream_skip[t][p]
 * (analysis.cpp:73-98) — and the original run's final images differ from it only
 * at the listed positions.  The regions are generated on the GPU (no region
 * crosses PCIe); otherwise equivalent to atc_testsets_upload_async. */
typedef struct {
  int32_t n_tests, n_ints, n_ptrs;
  const int64_t* int_values;   /* [T][n_ints]                                         */
  const int32_t* ptr_is_f32;   /* [n_ptrs]                                            */
  const int64_t* region_len;   /* [n_ptrs]                                            */
  const int32_t* test_ok;      /* [T]                                                 */
  const uint64_t* stream_seed; /* [T]: Rng seed of test t                             */
  const uint64_t* stream_skip; /* [T][n_ptrs]: draws before region p's first element  */
  const int64_t* diff_off;     /* [T*n_ptrs + 1]: entries of (t, p) = [off[i], off[i+1]) */
  const int32_t* diff_pos;     /* final-minus-init positions                           */
  const double* diff_val;      /* final values there                                  */
  /* nonzero: generate only the part of each region an evaluation can read.  With
   * U = test t's largest int value, every index the gemm / conv2d semantics read
   * for a binding that passes run_dispatch's extent check and the UB check is
   * below U^4 + 2U^2 + 2U + 1 (conv input: (N*C - 1)*H*W + (OH + R - 2)*W + OW + S - 2;
   * weights, outputs and every gemm operand are smaller), so region (t, p) is
   * generated up to that bound or one past its last final-minus-init position,
   * whichever is larger (capped at the region length).  Evaluations are unchanged;
   * atc_testsets_download refuses such a handle. */
  int32_t needed_only;
} atc_seeded_testsets;
int atc_testsets_upload_seeded(atc_ctx* ctx, const atc_seeded_testsets* ts, atc_testset_handle** out);

/* The recorded test sets when the caller already holds the probe images (the
 * liftc host builds them for its own original runs, rewriter.cpp:242-247): the
 * full host regions plus the original run's final-minus-init entries, of which
 * only what an evaluation can read crosses PCIe — region (t, p)'s prefix up to the
 * needed_only bound of the seeded form — U^4 + 2U^2 + 2U + 1, or one past its
 * last final-minus-init position — and the final images are rebuilt on the
 * device.  Evaluations are unchanged; atc_testsets_download refuses such a handle.
 * Host buffers are not retained (the prefixes are staged before returning). */
typedef struct {
  int32_t n_tests, n_ints, n_ptrs;
  const int64_t* int_values;   /* [T][n_ints]                                         */
  const int32_t* ptr_is_f32;   /* [n_ptrs]                                            */
  const int64_t* region_len;   /* [n_ptrs]                                            */
  const int32_t* test_ok;      /* [T]                                                 */
  const double* const* init;   /* [T*n_ptrs]: probe regions (NULL where test_ok[t] == 0) */
  const int64_t* diff_off;     /* [T*n_ptrs + 1]                                      */
  const int32_t* diff_pos;
  const double* diff_val;
} atc_prefix_testsets;
int atc_testsets_upload_prefix(atc_ctx* ctx, const atc_prefix_testsets* ts, atc_testset_handle** out);

/* New seeded contents for an existing handle (same n_tests, n_ints, n_ptrs,
 * region lengths and element types), written in place after every evaluation
 * already queued on the context's stream: prepared batches (atc_enum_batch_*)
 * over the handle stay valid and pick the new contents up on their next run. */
int atc_testsets_update_seeded(atc_ctx* ctx, atc_testset_handle* h, const atc_seeded_testsets* ts);
/* The same for n handles at once (handles[i] gets ts[i]); one ordering event for
 * all of them. */
int atc_testsets_update_seeded_many(atc_ctx* ctx, atc_testset_handle* const* handles,
                                    const atc_seeded_testsets* ts, int32_t n);

/* Copies a handle's regions back ((t, pointer) regions back to back, unpadded;
 * either pointer may be NULL) — for checks and debugging. */
int atc_testsets_download(atc_ctx* ctx, const atc_testset_handle* h, double* init, double* final_);

/* Explicit candidate list (ranked order).  arr_map[b*n_arrays + a] = user pointer
 * index bound to API array a; size_map[b*n_sizes + q] = user int index bound to
 * API size param q.  Outputs (host): fail_t[b] = first failing test or -1,
 * reason[b] = ATC_*; *first_pass = smallest b with reason ATC_PASS, or -1. */
int atc_eval_bindings(atc_ctx* ctx, const atc_spec_desc* spec, const atc_testset_handle* ts,
                      const uint8_t* arr_map, const uint8_t* size_map, int64_t n_bindings,
                      int32_t mode, int8_t* fail_t, int8_t* reason, int64_t* first_pass);

/* Several explicit lists at once — e.g. every spec's ranked candidates of one user
 * function (the specs pipeline.cpp:227-312 tries in turn), each against its own
 * test-set handle: one H2D of all maps, every list's kernels queued back to back,
 * one D2H and one synchronisation.  Each job's outputs equal atc_eval_bindings on
 * that job alone; status is ATC_OK or the job's own error (the call then returns
 * the first failing status). */
typedef struct atc_bind_job {
  const atc_spec_desc* spec;
  const atc_testset_handle* ts;
  const uint8_t* arr_map;   /* [n_bindings][spec->n_arrays] */
  const uint8_t* size_map;  /* [n_bindings][spec->n_sizes]  */
  int64_t n_bindings;
  int8_t* fail_t;           /* out [n_bindings] */
  int8_t* reason;           /* out [n_bindings] */
  int64_t first_pass;       /* out: smallest passing b, or -1 */
  int32_t status;           /* out */
} atc_bind_job;
int atc_eval_bindings_many(atc_ctx* ctx, atc_bind_job* jobs, int32_t n_jobs, int32_t mode);

/* Same with device-resident inputs/outputs on the caller's CUDA stream (cudaStream_t
 * passed as void*); returns without synchronising. */
int atc_eval_bindings_device(atc_ctx* ctx, const atc_spec_desc* spec, const atc_testset_handle* ts,
                             const uint8_t* d_arr_map, const uint8_t* d_size_map, int64_t n_bindings,
                             int32_t mode, int8_t* d_fail_t, int8_t* d_reason, void* stream);

/* Unpruned space in SURVEY.md Appendix C order: index = perm * n_ints^n_sizes + s,
 * API size param q bound to user int (s / n_ints^q) % n_ints; perms[p*n_arrays + a]
 * is the user pointer of API array a under permutation p.  Evaluates [begin, end)
 * and returns the passing indices (ascending, at most cap), their total count and a
 * histogram of first-failure reasons. */
int atc_eval_enumerated(atc_ctx* ctx, const atc_spec_desc* spec, const atc_testset_handle* ts,
                        const uint8_t* perms, int32_t n_perms, uint64_t begin, uint64_t end,
                        int32_t mode, uint64_t* survivors, int64_t cap, int64_t* n_survivors,
                        int64_t* reason_counts);

/* Many enumerated spaces in one stream pass (a corpus sweep: every function x
 * spec the pipeline would try).  No reference counterpart — it batches what
 * pipeline.cpp:248-310 does one spec at a time; each job's outputs equal
 * atc_eval_enumerated on that job alone.  All jobs' kernels are queued back to
 * back and the results come back in one copy; a job whose survivors or passing
 * list overflow the batched buffers is re-run through atc_eval_enumerated. */
typedef struct atc_enum_job {
  const atc_spec_desc* spec;
  const atc_testset_handle* ts;
  const uint8_t* perms;
  int32_t n_perms;
  uint64_t begin, end;
  uint64_t* survivors; /* out: ascending passing indices, at most cap */
  int64_t cap;
  int64_t n_survivors;                      /* out */
  int64_t reason_counts[ATC_REASON_COUNT];  /* out */
  int32_t status;                           /* out: ATC_OK or the job's error */
} atc_enum_job;
int atc_eval_enumerated_many(atc_ctx* ctx, atc_enum_job* jobs, int32_t n_jobs, int32_t mode);

/* The same sweep prepared once and run many times: create plans every job and
 * keeps its permutations on the device (jobs[] and the test-set handles must
 * outlive the batch); run evaluates every job and fills its outputs — eagerly on
 * the first run (and while profiling), afterwards as one CUDA-graph launch.
 * create returns NULL on error (atc_last_error). */
typedef struct atc_enum_batch atc_enum_batch;
atc_enum_batch* atc_enum_batch_create(atc_ctx* ctx, atc_enum_job* jobs, int32_t n_jobs, int32_t mode);
int atc_enum_batch_run(atc_ctx* ctx, atc_enum_batch* batch);
void atc_enum_batch_destroy(atc_ctx* ctx, atc_enum_batch* batch);

/* FP64 reference semantics on the GPU (equivalence::run_reference).  sizes[q] per
 * spec size param; buffers[a] (host, length buffer_len[a]) per spec array;
 * non-LiveIn arrays are rewritten in place. */
int atc_run_reference(atc_ctx* ctx, const atc_spec_desc* spec, const int64_t* sizes,
                      double* const* buffers, const int64_t* buffer_len);

/* make_oracle_dispatch handler body (rewriter.cpp:99-162) for one call whose
 * arguments are already decoded positionally: sizes[q] (ints), regions[a] with
 * region_len[a] and region_is_f32[a].  Returns ATC_ERR_DISPATCH with the
 * reference's message ("... is not positive" / "holds N elements, call needs M")
 * when run_dispatch would throw. */
int atc_dispatch(atc_ctx* ctx, const atc_spec_desc* spec, const int64_t* sizes,
                 double* const* regions, const int64_t* region_len, const int32_t* region_is_f32);

/* ---- Extended semantics (no reference counterpart) ------
 * The wide GEMM (transA/transB, alpha/beta, lda/ldb/ldc) and conv2d with stride,
 * padding and dilation that BASELINE configs 3-4 name.  The reference cannot
 * express them: run_dispatch ignores float scalars (rewriter.cpp:130-132) and its
 * conv2d is valid-padding, unit-stride (equivalence.cpp:67-93); its specs carry
 * size roles only.  The semantics are defined here (paper_2301_11659_b200/specs/
 * gemm_ext.json, conv2d_ext.json) and restated literally on the CPU in
 * oracle/ext_oracle.c, which known-answer vectors pin (tests/golden/
 * ext_known_answers.json) — parity against the reference is not defined.
 *
 *  gemm_ext (row-major): reason 2 ("dispatch failed") unless m, n, k, lda, ldb, ldc >= 1,
 *    transa, transb in {0, 1}, lda >= (ta ? m : k), ldb >= (tb ? k : n), ldc >= n and
 *    every footprint fits its region: ((ta ? k : m) - 1)*lda + (ta ? m : k) <= len(A),
 *    ((tb ? n : k) - 1)*ldb + (tb ? k : n) <= len(B), (m - 1)*ldc + n <= len(C).  Then
 *    for i < m, j < n: acc = sum_p opA(i,p)*opB(p,j) (p ascending, FP64, no FMA),
 *    opA(i,p) = ta ? A[p*lda + i] : A[i*lda + p], opB(p,j) = tb ? B[j*ldb + p] : B[p*ldb + j];
 *    C[i*ldc + j] = beta == 0 ? alpha*acc : alpha*acc + beta*C[i*ldc + j] (alpha 1 and
 *    beta 0 when the spec has no such role; f32 regions rounded at write-back).
 *  conv2d_ext (NCHW / KCRS): reason 2 unless n, c, h, w, k, r, s, stride_h/w, dil_h/w >= 1,
 *    pad_h/w >= 0, eh = h + 2*pad_h - dil_h*(r - 1) - 1 >= 0 (ew likewise), the bound
 *    oh / ow equal eh/stride_h + 1 / ew/stride_w + 1 (derived when the spec has no such
 *    role) and n*c*h*w <= len(in), k*c*r*s <= len(weights), n*k*oh*ow <= len(out).  Then
 *    out[b,q,y,x] = sum over z < c, u < r, v < s (ascending) of in[b,z,iy,ix]*wt[q,z,u,v],
 *    iy = y*stride_h - pad_h + u*dil_h, ix = x*stride_w - pad_w + v*dil_w, terms with iy
 *    or ix outside the image skipped (zero padding); stride/pad/dil default 1/0/1.
 *  P2 predicate per test t: reason 3 if test t's set failed, 2 as above, else 1 iff
 *  the full region of a non-LiveIn bound array differs from the recorded final
 *  (rewriter.cpp:264-279 tolerances), else the next t.
 *
 * Bindings: arrays as before; a size param binds a user int (size_map entry < n_ints)
 * or, for params with a constant domain (trans, stride, pad, dil), a constant
 * (entry n_ints + c selects iconst[c]); a float param binds a user float (entry <
 * the test sets' n_floats) or a constant (entry n_floats + c selects fconst[c]). */
enum { ATC_SEM_GEMM_EXT = 2, ATC_SEM_CONV2D_EXT = 3 };
enum { ATC_XR_TRANSA = 0, ATC_XR_TRANSB, ATC_XR_STRIDE_H, ATC_XR_STRIDE_W, ATC_XR_PAD_H, ATC_XR_PAD_W,
       ATC_XR_DIL_H, ATC_XR_DIL_W, ATC_XR_COUNT };
enum { ATC_FR_ALPHA = 0, ATC_FR_BETA = 1, ATC_FR_COUNT = 2 };
#define ATC_MAX_FLOATS 4
#define ATC_MAX_CONSTS 8
typedef struct {
  atc_spec_desc base;                    /* semantics ATC_SEM_*_EXT; arrays, sizes, base roles */
  int32_t n_floats;                      /* float params of the spec (spec order)              */
  int32_t ext_role_size[ATC_XR_COUNT];   /* size-param index of each extended role, -1 absent  */
  int32_t role_float[ATC_FR_COUNT];      /* float-param index of alpha / beta, -1 absent       */
  int32_t n_iconst, n_fconst;
  int64_t iconst[ATC_MAX_CONSTS];
  double fconst[ATC_MAX_CONSTS];
} atc_spec_ext;

/* Explicit candidate list under an extended spec: arr_map [n][n_arrays], size_map
 * [n][n_sizes], float_map [n][n_floats] (encodings above).  Outputs as
 * atc_eval_bindings (FP64, exact). */
int atc_eval_bindings_ext(atc_ctx* ctx, const atc_spec_ext* spec, const atc_testset_handle* ts,
                          const uint8_t* arr_map, const uint8_t* size_map, const uint8_t* float_map,
                          int64_t n_bindings, int8_t* fail_t, int8_t* reason, int64_t* first_pass);
/* The extended semantics on caller buffers (spec order): sizes[q] per size param,
 * floats[f] per float param, buffers[a] of buffer_len[a] doubles (non-LiveIn arrays
 * rewritten in place, f32-rounded where buffer_is_f32[a]).  ATC_ERR_DISPATCH (with
 * the failed check in atc_last_error) where the P2 predicate gives reason 2. */
int atc_run_reference_ext(atc_ctx* ctx, const atc_spec_ext* spec, const int64_t* sizes, const double* floats,
                          double* const* buffers, const int64_t* buffer_len, const int32_t* buffer_is_f32);

/* ---- Device groups --------------------------------------
 * Several GPUs of one process: one context (streams, scratch, pools) per device.
 * The candidate space shards naturally — an enumerated range is cut into
 * contiguous pieces (atc_plan_shards), each device evaluates its pieces against
 * its own replica of the recorded test sets, and the per-device results (passing
 * indices, reason histograms, first passing index) are combined: MIN of the first
 * passing index — the candidate the reference's rank-order loop (pipeline.cpp:
 * 248-310) reaches first —, SUM of the histograms, the ordered union of the
 * passing lists.  No data-path exchange: the devices run concurrently (one host
 * thread each) and only their result blocks come back.  A device may be listed
 * more than once (independent contexts on it). */
typedef struct atc_group atc_group;
typedef struct atc_group_testsets atc_group_testsets;
/* devices[i] for i < n (NULL: devices 0..n-1; n <= 0: every visible device).
 * Returns NULL only on allocation failure; check atc_group_last_error. */
atc_group* atc_group_create(const int32_t* devices, int32_t n);
void atc_group_destroy(atc_group* g);
const char* atc_group_last_error(const atc_group* g);
int32_t atc_group_size(const atc_group* g);
atc_ctx* atc_group_member(atc_group* g, int32_t i);   /* e.g. one per pipeline worker */
/* The same recorded test sets on every member device (as atc_testsets_upload_seeded /
 * _prefix, asynchronous). */
int atc_group_testsets_upload_seeded(atc_group* g, const atc_seeded_testsets* ts, atc_group_testsets** out);
int atc_group_testsets_upload_prefix(atc_group* g, const atc_prefix_testsets* ts, atc_group_testsets** out);
int atc_group_testsets_free(atc_group* g, atc_group_testsets* h);
const atc_testset_handle* atc_group_testsets_member(const atc_group_testsets* h, int32_t i);

typedef struct atc_group_job {
  const atc_spec_desc* spec;
  const atc_group_testsets* ts;
  const uint8_t* perms;
  int32_t n_perms;
  uint64_t begin, end;
  uint64_t* survivors;                      /* out: ascending passing indices, at most cap */
  int64_t cap;
  int64_t n_survivors;                      /* out: passing count (all devices)            */
  int64_t reason_counts[ATC_REASON_COUNT];  /* out: summed over devices                    */
  int64_t first_pass;                       /* out: smallest passing index, -1 if none     */
  int32_t status;                           /* out                                         */
} atc_group_job;
/* Every job's range sharded over the members (atc_plan_shards over the jobs' range
 * sizes), each member's share evaluated as one atc_eval_enumerated_many, then
 * combined.  Each job's outputs equal atc_eval_enumerated on one device. */
int atc_group_eval_enumerated_many(atc_group* g, atc_group_job* jobs, int32_t n_jobs, int32_t mode);
/* The same prepared once (each member an atc_enum_batch over its share, replayed as
 * one CUDA graph per device) and run many times. */
typedef struct atc_group_batch atc_group_batch;
atc_group_batch* atc_group_batch_create(atc_group* g, atc_group_job* jobs, int32_t n_jobs, int32_t mode);
int atc_group_batch_run(atc_group* g, atc_group_batch* b);
void atc_group_batch_destroy(atc_group* g, atc_group_batch* b);

/* The shard plan (host arithmetic, no device needed): rank r of `world` evaluates
 * [begin[r*n_jobs + j], end[r*n_jobs + j]) of job j (relative to the job's range;
 * empty when begin == end).  Spaces of >= 2^24 bindings are balanced with a
 * per-space cost model (a fixed part per piece plus a part per binding): largest
 * first, whole to the least-loaded rank when that stays within the per-rank target
 * (+15%), else in the fewest contiguous ~equal pieces that do; smaller spaces go
 * whole to one rank each, round-robin.  Deterministic: every rank computes the
 * same plan (paper_2301_11659_b200/workloads.py::plan_shards is the same rule). */
int atc_plan_shards(const uint64_t* counts, int32_t n_jobs, int32_t world, uint64_t* begin, uint64_t* end);

/* Backends.  precision: 0 = TF32 (1 pass), 1 = 3xTF32 (split, ~FP32 accuracy). */
enum { ATC_PREC_TF32 = 0, ATC_PREC_3XTF32 = 1 };
int atc_sgemm_rm(atc_ctx* ctx, const float* A, const float* B, float* C,
                 int64_t m, int64_t n, int64_t k, int32_t precision);
int atc_sgemm_rm_device(atc_ctx* ctx, const float* dA, const float* dB, float* dC,
                        int64_t m, int64_t n, int64_t k, int32_t precision, void* stream);
int atc_conv2d_nchw(atc_ctx* ctx, const float* in, const float* w, float* out, int64_t n, int64_t c,
                    int64_t h, int64_t w_, int64_t k, int64_t r, int64_t s, int32_t precision);
int atc_conv2d_nchw_device(atc_ctx* ctx, const float* d_in, const float* d_w, float* d_out,
                           int64_t n, int64_t c, int64_t h, int64_t w_, int64_t k, int64_t r,
                           int64_t s, int32_t precision, void* stream);

/* Host helpers for building P2 probe images exactly like analysis::build_probe_image
 * (analysis.cpp:73-98) on the std::mt19937_64 stream of liftc::Rng (rng.hpp:13-48):
 * skip `skip` raw draws of mt19937_64(seed), then write n raw draws / n values of
 * uniform_real(lo, hi), optionally rounded through float. */
void atc_mt64_raw(uint64_t seed, uint64_t skip, int64_t n, uint64_t* out);
void atc_mt64_uniform(uint64_t seed, uint64_t skip, int64_t n, double lo, double hi,
                      int32_t round_f32, double* out);

#ifdef __cplusplus
}
#endif
#endif /* ATC_B200_H */
