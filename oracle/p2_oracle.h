/* p2_oracle.h — CPU restatement of the reference's hot path (TEST INFRASTRUCTURE).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library, and only as the checker.  Every function cites the reference
 * code it restates (paths relative to /root/reference/proj).
 *
 * Parity pins (tests/test_oracle.py): the frozen vectors of
 * tests/equivalence_test.cpp:76-121 and the per-binding verify_rewrite verdicts
 * dumped from the compiled reference (oracle/_ref/ref_tool golden) for every
 * GEMM/conv corpus program.
 */
#ifndef P2_ORACLE_H
#define P2_ORACLE_H
#include <stdint.h>

/* Spec decode (api_spec.hpp:26-66); same field meaning as atc_spec_desc. */
typedef struct {
  int32_t semantics; /* 0 gemm, 1 conv2d */
  int32_t layout;    /* 0 row, 1 col */
  int32_t n_arrays, n_sizes;
  int32_t array_role[4];
  int32_t array_livein[4];
  int32_t array_ndims[4];
  int32_t array_dims[4][6];
  int32_t role_size[15];
} oracle_spec;

/* equivalence::run_reference (equivalence.cpp:131-139): gemm :40-65 or conv2d
 * :67-93 over caller buffers indexed by API array (spec order), output rewritten
 * in place.  Returns 0, or -1 if any access would leave a buffer (UB in the
 * reference). */
int oracle_run_reference(const oracle_spec* s, const int64_t* sizes, double* const* bufs, const int64_t* lens);

/* One binding against recorded test sets, exactly as verify_rewrite does it
 * (rewriter.cpp:235-281): per t, run_dispatch's checks (:136-148) -> reason 2,
 * full-region copies, run_reference, write-back with f32 rounding (:152-161),
 * compare of the full region of every non-LiveIn bound array (:264-279) ->
 * reason 1; test sets whose draw/original run failed -> reason 3.  Writes the
 * first failing t (or -1) and the reason (0 pass). */
void oracle_verify_binding(const oracle_spec* s, int T, int nI, int nP, const int64_t* ints,
                           const int32_t* is_f32, const int64_t* region_len, const double* const* init,
                           const double* const* fin, const int32_t* test_ok, const uint8_t* arr_map,
                           const uint8_t* size_map, int8_t* fail_t, int8_t* reason);

/* The same over n bindings with `threads` host threads. */
void oracle_verify_many(const oracle_spec* s, int T, int nI, int nP, const int64_t* ints, const int32_t* is_f32,
                        const int64_t* region_len, const double* const* init, const double* const* fin,
                        const int32_t* test_ok, const uint8_t* arr_map, const uint8_t* size_map, int64_t n,
                        int threads, int8_t* fail_t, int8_t* reason);

/* profitability::cpu_gemm (profitability.cpp:14-21) and xpu_gemm (:25-63). */
void oracle_cpu_gemm(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k);
void oracle_xpu_gemm(const float* a, const float* b, float* c, int64_t m, int64_t n, int64_t k, int threads);

/* ---- Extended semantics (include/atc_b200.h, "Extended semantics") -----------
 * No reference counterpart: oracle/ext_oracle.c IS the definition, restated
 * literally (full-region copies, the loops as written in the header comment, full
 * compares); pinned by the hand-derived known answers of
 * tests/golden/ext_known_answers.json (tests/test_ext.py). */
typedef struct {
  oracle_spec base;       /* semantics 2 gemm_ext, 3 conv2d_ext */
  int32_t n_floats;
  int32_t ext_role_size[8];
  int32_t role_float[2];
  int32_t n_iconst, n_fconst;
  int64_t iconst[8];
  double fconst[8];
} oracle_spec_ext;

/* Runs the extended semantics on caller buffers; returns 0, or 2 when the dispatch
 * checks fail (buffers untouched).  detail (optional, >= 128 bytes) names the check. */
int oracle_run_ext(const oracle_spec_ext* s, const int64_t* sizes, const double* floats, double* const* bufs,
                   const int64_t* lens, const int32_t* is_f32, char* detail);

/* One extended binding against recorded test sets (the P2 predicate of the header);
 * floats: [T][nF] user float values. */
void oracle_verify_ext_many(const oracle_spec_ext* s, int T, int nI, int nP, int nF, const int64_t* ints,
                            const double* floats, const int32_t* is_f32, const int64_t* region_len,
                            const double* const* init, const double* const* fin, const int32_t* test_ok,
                            const uint8_t* arr_map, const uint8_t* size_map, const uint8_t* float_map, int64_t n,
                            int threads, int8_t* fail_t, int8_t* reason);

/* FNV-1a 64 over raw bytes (pins regenerated probe regions to the golden dump). */
uint64_t oracle_fnv1a(const void* p, int64_t nbytes);

#endif
