/* ext_oracle.c — CPU statement of the extended semantics (TEST INFRASTRUCTURE).
 *
 * gemm_ext (transA/transB, alpha/beta, lda/ldb/ldc) and conv2d_ext (stride,
 * padding, dilation) have no counterpart in the reference (rewriter.cpp:130-132
 * ignores float scalars; equivalence.cpp:67-93 is valid/unit-stride only), so this
 * file is their definition — the rules of include/atc_b200.h ("Extended
 * semantics"), written as plain loops over full-region copies like
 * oracle_verify_binding (p2_oracle.c), which restates verify_rewrite
 * (rewriter.cpp:235-281).  Parity against the reference is not defined; the
 * known answers of tests/golden/ext_known_answers.json (hand-derived, exact binary
 * fractions) pin it (tests/test_ext.py), and the GPU path is checked against it.
 * Only tests/ may load it (liboracle_p2.so).
 */
#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "p2_oracle.h"

enum { SZ_M = 0, SZ_N, SZ_K, SZ_LDA, SZ_LDB, SZ_LDC, SZ_CN, SZ_CC, SZ_CH, SZ_CW, SZ_CK, SZ_CR, SZ_CS, SZ_COH, SZ_COW };
enum { XR_TA = 0, XR_TB, XR_SH, XR_SW, XR_PH, XR_PW, XR_DH, XR_DW };

static int64_t base_role(const oracle_spec_ext* s, const int64_t* sizes, int role, int64_t fb) {
  const int q = s->base.role_size[role];
  return q >= 0 ? sizes[q] : fb;
}
static int64_t ext_role(const oracle_spec_ext* s, const int64_t* sizes, int role, int64_t fb) {
  const int q = s->ext_role_size[role];
  return q >= 0 ? sizes[q] : fb;
}
static double float_role(const oracle_spec_ext* s, const double* floats, int role, double fb) {
  const int f = s->role_float[role];
  return f >= 0 ? floats[f] : fb;
}
static int array_of_role(const oracle_spec_ext* s, int role) {
  for (int a = 0; a < s->base.n_arrays; ++a)
    if (s->base.array_role[a] == role) return a;
  return -1;
}
static int fail(char* detail, const char* msg) {
  if (detail) snprintf(detail, 128, "%s", msg);
  return 2;
}

static int run_gemm_ext(const oracle_spec_ext* s, const int64_t* sz, const double* fl, double* const* bufs,
                        const int64_t* lens, const int32_t* is_f32, char* detail) {
  const int64_t m = base_role(s, sz, SZ_M, 0), n = base_role(s, sz, SZ_N, 0), k = base_role(s, sz, SZ_K, 0);
  const int64_t lda = base_role(s, sz, SZ_LDA, 0), ldb = base_role(s, sz, SZ_LDB, 0), ldc = base_role(s, sz, SZ_LDC, 0);
  const int64_t ta = ext_role(s, sz, XR_TA, 0), tb = ext_role(s, sz, XR_TB, 0);
  const double alpha = float_role(s, fl, 0, 1.0), beta = float_role(s, fl, 1, 0.0);
  const int aA = array_of_role(s, 0), aB = array_of_role(s, 1), aC = array_of_role(s, 2);
  if (m < 1 || n < 1 || k < 1 || lda < 1 || ldb < 1 || ldc < 1) return fail(detail, "size is not positive");
  if ((ta != 0 && ta != 1) || (tb != 0 && tb != 1)) return fail(detail, "transpose flag is not 0 or 1");
  if (lda < (ta ? m : k) || ldb < (tb ? k : n) || ldc < n) return fail(detail, "leading dimension too small");
  if (((ta ? k : m) - 1) * lda + (ta ? m : k) > lens[aA]) return fail(detail, "A footprint exceeds its region");
  if (((tb ? n : k) - 1) * ldb + (tb ? k : n) > lens[aB]) return fail(detail, "B footprint exceeds its region");
  if ((m - 1) * ldc + n > lens[aC]) return fail(detail, "C footprint exceeds its region");
  const double* A = bufs[aA];
  const double* B = bufs[aB];
  double* C = bufs[aC];
  for (int64_t i = 0; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int64_t p = 0; p < k; ++p) {
        const double av = ta ? A[p * lda + i] : A[i * lda + p];
        const double bv = tb ? B[j * ldb + p] : B[p * ldb + j];
        acc += av * bv;
      }
      double out;
      if (beta == 0.0) {
        out = alpha * acc;
      } else {
        const double t1 = alpha * acc, t2 = beta * C[i * ldc + j];
        out = t1 + t2;
      }
      C[i * ldc + j] = is_f32 && is_f32[aC] ? (double)(float)out : out;
    }
  return 0;
}

static int run_conv_ext(const oracle_spec_ext* s, const int64_t* sz, double* const* bufs, const int64_t* lens,
                        const int32_t* is_f32, char* detail) {
  const int64_t N = base_role(s, sz, SZ_CN, 0), C = base_role(s, sz, SZ_CC, 0), H = base_role(s, sz, SZ_CH, 0);
  const int64_t W = base_role(s, sz, SZ_CW, 0), K = base_role(s, sz, SZ_CK, 0), R = base_role(s, sz, SZ_CR, 0);
  const int64_t S = base_role(s, sz, SZ_CS, 0);
  const int64_t sh = ext_role(s, sz, XR_SH, 1), sw = ext_role(s, sz, XR_SW, 1);
  const int64_t ph = ext_role(s, sz, XR_PH, 0), pw = ext_role(s, sz, XR_PW, 0);
  const int64_t dh = ext_role(s, sz, XR_DH, 1), dw = ext_role(s, sz, XR_DW, 1);
  const int aI = array_of_role(s, 0), aW = array_of_role(s, 1), aO = array_of_role(s, 2);
  if (N < 1 || C < 1 || H < 1 || W < 1 || K < 1 || R < 1 || S < 1) return fail(detail, "size is not positive");
  if (sh < 1 || sw < 1 || dh < 1 || dw < 1 || ph < 0 || pw < 0) return fail(detail, "bad stride / dilation / padding");
  const int64_t eh = H + 2 * ph - dh * (R - 1) - 1, ew = W + 2 * pw - dw * (S - 1) - 1;
  if (eh < 0 || ew < 0) return fail(detail, "filter larger than the padded image");
  const int64_t oh_x = eh / sh + 1, ow_x = ew / sw + 1;
  const int64_t OH = base_role(s, sz, SZ_COH, oh_x), OW = base_role(s, sz, SZ_COW, ow_x);
  if (OH != oh_x || OW != ow_x) return fail(detail, "output size does not match stride / padding / dilation");
  if (N * C * H * W > lens[aI] || K * C * R * S > lens[aW] || N * K * OH * OW > lens[aO])
    return fail(detail, "extent exceeds its region");
  const double* in = bufs[aI];
  const double* wt = bufs[aW];
  double* out = bufs[aO];
  for (int64_t b = 0; b < N; ++b)
    for (int64_t q = 0; q < K; ++q)
      for (int64_t y = 0; y < OH; ++y)
        for (int64_t x = 0; x < OW; ++x) {
          double acc = 0.0;
          for (int64_t z = 0; z < C; ++z)
            for (int64_t u = 0; u < R; ++u)
              for (int64_t v = 0; v < S; ++v) {
                const int64_t iy = y * sh - ph + u * dh, ix = x * sw - pw + v * dw;
                if (iy < 0 || iy >= H || ix < 0 || ix >= W) continue;
                acc += in[((b * C + z) * H + iy) * W + ix] * wt[((q * C + z) * R + u) * S + v];
              }
          const int64_t o = ((b * K + q) * OH + y) * OW + x;
          out[o] = is_f32 && is_f32[aO] ? (double)(float)acc : acc;
        }
  return 0;
}

int oracle_run_ext(const oracle_spec_ext* s, const int64_t* sizes, const double* floats, double* const* bufs,
                   const int64_t* lens, const int32_t* is_f32, char* detail) {
  if (s->base.semantics == 2) return run_gemm_ext(s, sizes, floats, bufs, lens, is_f32, detail);
  if (s->base.semantics == 3) return run_conv_ext(s, sizes, bufs, lens, is_f32, detail);
  if (detail) snprintf(detail, 128, "no extended semantics %d", s->base.semantics);
  return -1;
}

static void verify_ext(const oracle_spec_ext* s, int T, int nI, int nP, int nF, const int64_t* ints,
                       const double* floats, const int32_t* is_f32, const int64_t* region_len,
                       const double* const* init, const double* const* fin, const int32_t* test_ok,
                       const uint8_t* arr_map, const uint8_t* size_map, const uint8_t* float_map, int8_t* fail_t,
                       int8_t* reason) {
  double* bufs[4] = {0, 0, 0, 0};
  int64_t lens[4] = {0, 0, 0, 0};
  int32_t f32[4] = {0, 0, 0, 0};
  int64_t sizes[16]; /* ATC_MAX_EXT_SIZES: conv2d_ext has 15 size params */
  double fl[4];
  *fail_t = -1;
  *reason = 0;
  for (int t = 0; t < T; ++t) {
    if (!test_ok[t]) {
      *fail_t = (int8_t)t;
      *reason = 3;
      goto done;
    }
    for (int q = 0; q < s->base.n_sizes; ++q)
      sizes[q] = size_map[q] < nI ? ints[(int64_t)t * nI + size_map[q]] : s->iconst[size_map[q] - nI];
    for (int f = 0; f < s->n_floats; ++f)
      fl[f] = float_map[f] < nF ? floats[(int64_t)t * nF + float_map[f]] : s->fconst[float_map[f] - nF];
    for (int a = 0; a < s->base.n_arrays; ++a) {  /* full-region copies */
      const int p = arr_map[a];
      lens[a] = region_len[p];
      f32[a] = is_f32[p];
      bufs[a] = (double*)realloc(bufs[a], (size_t)lens[a] * sizeof(double));
      memcpy(bufs[a], init[(int64_t)t * nP + p], (size_t)lens[a] * sizeof(double));
    }
    if (oracle_run_ext(s, sizes, fl, bufs, lens, f32, NULL) != 0) {
      *fail_t = (int8_t)t;
      *reason = 2;
      goto done;
    }
    for (int a = 0; a < s->base.n_arrays; ++a) {  /* full-region compare (rewriter.cpp:264-279) */
      if (s->base.array_livein[a]) continue;
      const int p = arr_map[a];
      const double rel = f32[a] ? 1e-4 : 1e-9, abs_ = f32[a] ? 1e-6 : 1e-12;
      const double* want = fin[(int64_t)t * nP + p];
      for (int64_t i = 0; i < lens[a]; ++i)
        if (fabs(bufs[a][i] - want[i]) > abs_ + rel * fabs(want[i])) {
          *fail_t = (int8_t)t;
          *reason = 1;
          goto done;
        }
    }
  }
done:
  for (int a = 0; a < 4; ++a) free(bufs[a]);
}

typedef struct {
  const oracle_spec_ext* s;
  int T, nI, nP, nF;
  const int64_t* ints;
  const double* floats;
  const int32_t* is_f32;
  const int64_t* region_len;
  const double* const* init;
  const double* const* fin;
  const int32_t* test_ok;
  const uint8_t *arr_map, *size_map, *float_map;
  int64_t n;
  int8_t *fail_t, *reason;
  atomic_llong next;
} ext_args;

static void* ext_worker(void* p) {
  ext_args* a = (ext_args*)p;
  for (;;) {
    const long long b = atomic_fetch_add(&a->next, 1);
    if (b >= a->n) break;
    verify_ext(a->s, a->T, a->nI, a->nP, a->nF, a->ints, a->floats, a->is_f32, a->region_len, a->init, a->fin,
               a->test_ok, a->arr_map + b * a->s->base.n_arrays, a->size_map + b * a->s->base.n_sizes,
               a->float_map + b * (a->s->n_floats > 0 ? a->s->n_floats : 0), a->fail_t + b, a->reason + b);
  }
  return NULL;
}

void oracle_verify_ext_many(const oracle_spec_ext* s, int T, int nI, int nP, int nF, const int64_t* ints,
                            const double* floats, const int32_t* is_f32, const int64_t* region_len,
                            const double* const* init, const double* const* fin, const int32_t* test_ok,
                            const uint8_t* arr_map, const uint8_t* size_map, const uint8_t* float_map, int64_t n,
                            int threads, int8_t* fail_t, int8_t* reason) {
  ext_args a = {s,       T,        nI,  nP,       nF,       ints,     floats, is_f32, region_len, init, fin,
                test_ok, arr_map, size_map, float_map, n, fail_t, reason, 0};
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t th[256];
  for (int i = 0; i < threads; ++i) pthread_create(&th[i], NULL, ext_worker, &a);
  for (int i = 0; i < threads; ++i) pthread_join(th[i], NULL);
}
