// C ABI: recorded P2 test sets on the device (uploads, seeded generation, in-place updates).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "atc_b200.h"
#include "capi_internal.h"

using namespace atc;

// Fills an allocated handle from full host regions (`ts_full`) or from seeds +
// final-minus-init entries (`sd`, regions generated on the device), on the
// handle's copy stream, and records its ready event.
// needed_only bound of region (t, p): max(U^4 + 2U^2 + 2U + 1, last final-minus-init
// position + 1), U = test t's largest int (include/atc_b200.h), capped at the region
// length; the whole region without needed_only.
static std::vector<int64_t> region_need(const atc_testset_handle* h, const atc_seeded_testsets* sd) {
  const int T = h->T, nI = h->nI, nP = h->nP;
  std::vector<int64_t> need((size_t)T * nP);
  for (int t = 0; t < T; ++t) {
    int64_t u = 1;
    for (int q = 0; q < nI; ++q) u = std::max<int64_t>(u, sd->int_values[(size_t)t * nI + q]);
    const int64_t bound = u > 46340 ? INT64_MAX : u * u * u * u + 2 * u * u + 2 * u + 1;
    for (int p = 0; p < nP; ++p) {
      const size_t i = (size_t)t * nP + p;
      int64_t n = bound;
      for (int64_t e = sd->diff_off[i]; e < sd->diff_off[i + 1]; ++e) n = std::max<int64_t>(n, sd->diff_pos[e] + 1);
      need[i] = sd->needed_only ? std::min<int64_t>(n, h->lens[p]) : h->lens[p];
    }
  }
  return need;
}

// The handle's metadata block (the TestsetView arrays) in host staging: ints, region
// lengths / offsets, dirty-list offsets, f32 flags, test_ok, floats; dirty counts 0
// and dirty_max -1 until the dirty lists are built.
static void fill_meta(const atc_testset_handle* h, const int64_t* int_values, const int32_t* test_ok,
                      const double* floats, uint8_t* meta) {
  const int T = h->T, nI = h->nI, nP = h->nP;
  const size_t TP = (size_t)T * nP;
  std::memset(meta, 0, h->meta_bytes);
  auto put = [&](size_t o, const void* src, size_t bytes) {
    if (bytes) std::memcpy(meta + o, src, bytes);
  };
  put(h->o_ints, int_values, (size_t)T * nI * 8);
  put(h->o_rlen, h->lens.data(), nP * 8);
  put(h->o_roff, h->off.data(), TP * 8);
  put(h->o_dof, h->doff.data(), TP * 8);
  put(h->o_isf, h->is_f32.data(), nP * 4);
  if (floats) put(h->o_flt, floats, (size_t)T * h->nF * 8);
  for (int t = 0; t < T; ++t) {
    const int32_t ok_t = test_ok ? (test_ok[t] ? 1 : 0) : 1;
    put(h->o_tok + t * 4, &ok_t, 4);
  }
  for (size_t i = 0; i < TP; ++i) {
    const int32_t neg = -1;
    put(h->o_dmax + i * 4, &neg, 4);  // dirty counts stay 0
  }
}

// pre (optional, with sd): the caller's own init regions [T*nP] — only their needed
// prefixes are staged and copied, instead of generating them from the seeds.
static int testsets_fill(atc_ctx* ctx, atc_testset_handle* h, const atc_testsets* ts_full,
                         const atc_seeded_testsets* sd, bool sync, bool pinned_staging = false,
                         cudaEvent_t reuse = nullptr, const double* const* pre = nullptr) {
  const int T = h->T, nI = h->nI, nP = h->nP;
  const size_t TP = (size_t)T * nP;
  const int64_t* int_values = ts_full ? ts_full->int_values : sd->int_values;
  const int32_t* test_ok = ts_full ? ts_full->test_ok : sd->test_ok;
  h->h_ints.assign(int_values, int_values + (size_t)T * nI);
  // every small array in one block, built in pinned staging and copied once; the
  // seeded block follows it in the same staging buffer
  const int64_t nd_s = sd ? sd->diff_off[TP] : 0;
  std::vector<int64_t> need = sd ? region_need(h, sd) : std::vector<int64_t>();
  if (pre)  // a failed test has no region: every binding fails there (reason 3), nothing to stage
    for (size_t i = 0; i < TP; ++i)
      if (!pre[i] || (test_ok && !test_ok[i / nP])) need[i] = 0;
  std::vector<int64_t> pre_off(pre ? TP + 1 : 0, 0);
  for (size_t i = 0; pre && i < TP; ++i)
    pre_off[i + 1] = pre_off[i] + need[i];
  const size_t pre_bytes = pre ? ((size_t)pre_off[TP] * 8 + 15) / 16 * 16 + ((TP + 1) * 8 + 15) / 16 * 16 : 0;
  const size_t seeded_need =
      sd ? ((size_t)T * 8 + 15) / 16 * 16 + (TP * 8 + 15) / 16 * 16 + ((TP + 1) * 8 + 15) / 16 * 16 +
               ((size_t)nd_s * 8 + 15) / 16 * 16 + ((size_t)nd_s * 4 + 15) / 16 * 16 + (TP * 8 + 15) / 16 * 16 +
               pre_bytes
         : 0;
  // in-place updates stage through the handle's pinned buffer (true async DMA,
  // allocated once); a first upload stages through pageable memory (the driver
  // copies it before returning) and avoids a pinned allocation per handle
  std::vector<uint8_t> pageable;
  uint8_t* meta = nullptr;
  if (pinned_staging) {
    if (h->ready && !atc_cuda_ok(ctx, cudaEventSynchronize(h->ready), "staging reuse"))  // previous DMA done
      return ATC_ERR_CUDA;
    if (h->pin_bytes < h->meta_bytes + seeded_need) {
      if (h->pin) cudaFreeHost(h->pin);
      h->pin = nullptr;
      h->pin_bytes = 0;
      if (!atc_cuda_ok(ctx, cudaMallocHost(&h->pin, h->meta_bytes + seeded_need), "cudaMallocHost"))
        return ATC_ERR_CUDA;
      h->pin_bytes = h->meta_bytes + seeded_need;
    }
    meta = h->pin;
  } else {
    pageable.resize(h->meta_bytes + seeded_need);
    meta = pageable.data();
  }
  fill_meta(h, int_values, test_ok, ts_full && h->nF ? ts_full->float_values : nullptr, meta);
  cudaStream_t st = ctx->copy_stream[h->cs];
  if (ctx->free_pending & (1ull << h->cs)) {  // pool memory freed by earlier handles
    cudaStreamWaitEvent(st, ctx->free_ev, 0);
    ctx->free_pending &= ~(1ull << h->cs);
  }
  if (reuse) cudaStreamWaitEvent(st, reuse, 0);  // in-place update: earlier readers first
  bool ok = atc_cuda_ok(ctx, cudaMemcpyAsync(h->meta, meta, h->meta_bytes, cudaMemcpyHostToDevice, st),
                        "H2D metadata");
  double* init = const_cast<double*>(h->view.init);
  double* fin = const_cast<double*>(h->view.fin);
  bool fused = false;  // dirty lists built by k_probe_regions
  if (ts_full) {
    // host regions that lie back to back in the same order as the device pool are
    // copied as one run (one DMA instead of T*n_ptrs)
    struct Run {
      const double* src = nullptr;
      size_t dst = 0, bytes = 0;
    };
    Run run_i, run_f;
    auto flush = [&](Run& r, double* base, const char* what) {
      if (r.bytes)
        ok = ok && atc_cuda_ok(ctx, cudaMemcpyAsync(base + r.dst, r.src, r.bytes, cudaMemcpyHostToDevice, st), what);
      r = Run{};
    };
    auto add = [&](Run& r, double* base, const double* src, size_t dst, size_t bytes, const char* what) {
      if (r.bytes && r.src + r.bytes / 8 == src && r.dst + r.bytes / 8 == dst && r.bytes % 256 == 0) {
        r.bytes += bytes;
        return;
      }
      flush(r, base, what);
      r.src = src;
      r.dst = dst;
      r.bytes = bytes;
    };
    for (int t = 0; t < T && ok; ++t)
      for (int p = 0; p < nP && ok; ++p) {
        const size_t i = (size_t)t * nP + p;
        const size_t bytes = (size_t)h->lens[p] * 8;
        const double* hi = ts_full->init[i];
        const double* hf = ts_full->final_[i];
        if (!hi || !hf) {
          // a test whose original run failed has no final image; the region stays
          // unused because every binding fails at t (test_ok[t] == 0)
          if (test_ok && test_ok[t]) {
            atc_set_error(ctx, "test %d pointer %d: missing region", t, p);
            ok = false;
          }
          ok = ok && atc_cuda_ok(ctx, cudaMemsetAsync(init + h->off[i], 0, bytes, st), "memset") &&
               atc_cuda_ok(ctx, cudaMemsetAsync(fin + h->off[i], 0, bytes, st), "memset");
          continue;
        }
        add(run_i, init, hi, (size_t)h->off[i], bytes, "H2D init");
        add(run_f, fin, hf, (size_t)h->off[i], bytes, "H2D final");
      }
    flush(run_i, init, "H2D init");
    flush(run_f, fin, "H2D final");
  } else if (ok) {
    // regions from the tests' mt19937_64 streams (k_probe_regions), then the
    // final-minus-init entries scattered into the final images (k_apply_diffs)
    const int64_t nd = sd->diff_off[TP];
    for (int64_t i = 0; ok && i < nd; ++i)
      if (sd->diff_pos[i] < 0) {
        atc_set_error(ctx, "negative final-minus-init position");
        ok = false;
      }
    size_t so = 0;
    auto take = [&](size_t bytes) {
      const size_t o = so;
      so += (bytes + 15) / 16 * 16;
      return o;
    };
    const size_t o_seeds = take((size_t)T * 8), o_skips = take(TP * 8), o_doffs = take((TP + 1) * 8),
                 o_dvs = take((size_t)nd * 8), o_dps = take((size_t)nd * 4), o_need = take(TP * 8);
    const size_t o_pre = pre ? take((size_t)pre_off[TP] * 8) : 0, o_preoff = pre ? take((TP + 1) * 8) : 0;
    h->needed_only = sd->needed_only != 0;
    if (ok && so > h->seeded_cap) {  // grow (the old block stays owned by the handle)
      h->seeded = (uint8_t*)atc_pool_alloc(ctx, std::max(so, (size_t)256));
      if (h->seeded) h->allocations.push_back(h->seeded);
      h->seeded_cap = h->seeded ? so : 0;
      if (!h->seeded) {
        atc_set_error(ctx, "device allocation failed (seeded test sets)");
        ok = false;
      }
    }
    if (ok) {
      uint8_t* sb = meta + h->meta_bytes;  // so == seeded_need
      std::memcpy(sb + o_seeds, sd->stream_seed, (size_t)T * 8);
      std::memcpy(sb + o_skips, sd->stream_skip, TP * 8);
      std::memcpy(sb + o_doffs, sd->diff_off, (TP + 1) * 8);
      if (nd) {
        std::memcpy(sb + o_dvs, sd->diff_val, (size_t)nd * 8);
        std::memcpy(sb + o_dps, sd->diff_pos, (size_t)nd * 4);
      }
      std::memcpy(sb + o_need, need.data(), TP * 8);
      if (pre) {
        for (size_t i = 0; i < TP; ++i)
          if (pre_off[i + 1] > pre_off[i])
            std::memcpy(sb + o_pre + (size_t)pre_off[i] * 8, pre[i], (size_t)(pre_off[i + 1] - pre_off[i]) * 8);
        std::memcpy(sb + o_preoff, pre_off.data(), (TP + 1) * 8);
      }
      ok = atc_cuda_ok(ctx, cudaMemcpyAsync(h->seeded, sb, so, cudaMemcpyHostToDevice, st), "H2D seeds");
    }
    if (ok) {
      const TestsetView& v = h->view;
      // needed_only: one kernel generates the prefixes, applies the diffs and builds
      // the dirty lists; else whole regions, then k_apply_diffs and k_build_dirty
      const int64_t* dn = sd->needed_only ? (const int64_t*)(h->seeded + o_need) : nullptr;
      k_probe_regions<<<T, kProbeThreads, 0, st>>>(T, nP, (const uint64_t*)(h->seeded + o_seeds),
                                         (const uint64_t*)(h->seeded + o_skips), v.region_len, v.is_f32,
                                         v.region_off, dn, init, fin, v, (const int64_t*)(h->seeded + o_doffs),
                                         (const int32_t*)(h->seeded + o_dps), (const double*)(h->seeded + o_dvs),
                                         pre ? (const double*)(h->seeded + o_pre) : nullptr,
                                         pre ? (const int64_t*)(h->seeded + o_preoff) : nullptr);
      if (!dn)
        k_apply_diffs<<<(unsigned)TP, 256, 0, st>>>(nP, v.region_len, v.region_off,
                                                    (const int64_t*)(h->seeded + o_doffs),
                                                    (const int32_t*)(h->seeded + o_dps),
                                                    (const double*)(h->seeded + o_dvs), fin);
      fused = dn != nullptr;
      ok = atc_cuda_ok(ctx, cudaGetLastError(), "k_probe_regions");
    }
  }
  if (ok) {
    if (!fused) {
      int64_t maxlen = 0;
      for (int p = 0; p < nP; ++p) maxlen = std::max<int64_t>(maxlen, h->lens[p]);
      dim3 grid((unsigned)std::min<int64_t>((maxlen + 255) / 256, 64), (unsigned)(T * nP));
      k_build_dirty<<<grid, 256, 0, st>>>(h->view, const_cast<int32_t*>(h->view.dirty_pos),
                                          const_cast<int32_t*>(h->view.dirty_cnt),
                                          const_cast<int32_t*>(h->view.dirty_max));
    }
    ok = atc_cuda_ok(ctx, cudaGetLastError(), "k_build_dirty") &&
         (h->ready || atc_cuda_ok(ctx, cudaEventCreateWithFlags(&h->ready, cudaEventDisableTiming), "cudaEventCreate")) &&
         atc_cuda_ok(ctx, cudaEventRecord(h->ready, st), "cudaEventRecord") &&
         (!sync || atc_cuda_ok(ctx, cudaEventSynchronize(h->ready), "upload sync"));
  }
  return ok ? ATC_OK : ATC_ERR_CUDA;
}

// Both upload forms: full host regions (`ts`) or seeds + final-minus-init entries
// (`sd`, regions generated on the device); the common header fields are equal.
static int testsets_upload(atc_ctx* ctx, const atc_testsets* ts_full, const atc_seeded_testsets* sd,
                           atc_testset_handle** out, bool sync, const double* const* pre = nullptr) {
  ATC_ENTER(ctx);
  atc_testsets hdr{};
  if (ts_full) hdr = *ts_full;
  if (sd) {
    hdr.n_tests = sd->n_tests;
    hdr.n_ints = sd->n_ints;
    hdr.n_ptrs = sd->n_ptrs;
    hdr.int_values = sd->int_values;
    hdr.ptr_is_f32 = sd->ptr_is_f32;
    hdr.region_len = sd->region_len;
    hdr.test_ok = sd->test_ok;
  }
  const atc_testsets* ts = &hdr;
  if ((!ts_full && !sd) || !out || ts->n_tests < 1 || ts->n_tests > kMaxT || ts->n_ints < 1 ||
      ts->n_ints > kMaxInts || ts->n_ptrs < 1 || ts->n_ptrs > kMaxPtrs || !ts->int_values || !ts->region_len ||
      !ts->ptr_is_f32 || (sd && (!sd->stream_seed || !sd->stream_skip || !sd->diff_off || sd->diff_off[0] != 0))) {
    atc_set_error(ctx, "malformed test sets");
    return ATC_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  const int T = ts->n_tests, nI = ts->n_ints, nP = ts->n_ptrs;
  const size_t TP = (size_t)T * nP;
  if (ts_full && (ts_full->n_floats < 0 || ts_full->n_floats > ATC_MAX_FLOATS ||
                  (ts_full->n_floats > 0 && !ts_full->float_values))) {
    atc_set_error(ctx, "malformed test sets (floats)");
    return ATC_ERR_ARG;
  }
  auto* h = new atc_testset_handle();
  h->T = T;
  h->nI = nI;
  h->nP = nP;
  h->nF = ts_full ? ts_full->n_floats : 0;
  h->lens.assign(ts->region_len, ts->region_len + nP);
  h->is_f32.assign(ts->ptr_is_f32, ts->ptr_is_f32 + nP);
  // region pool layout: (t, p) regions back to back, each 32-element aligned
  h->off.resize(TP);
  h->doff.resize(TP);
  int64_t total = 0, dtotal = 0;
  for (int t = 0; t < T; ++t)
    for (int p = 0; p < nP; ++p) {
      int64_t len = ts->region_len[p];
      if (len < 4 || len >= (1LL << 31)) {
        atc_set_error(ctx, "region %d length %lld outside [4, 2^31)", p, (long long)len);
        delete h;
        return ATC_ERR_ARG;
      }
      h->off[(size_t)t * nP + p] = total;
      h->doff[(size_t)t * nP + p] = dtotal;
      total += (len + 31) / 32 * 32;
      dtotal += len;
    }
  size_t mo = 0;
  auto take = [&](size_t bytes) {
    const size_t o = mo;
    mo += (bytes + 15) / 16 * 16;
    return o;
  };
  h->o_ints = take((size_t)T * nI * 8);
  h->o_rlen = take(nP * 8);
  h->o_roff = take(TP * 8);
  h->o_dof = take(TP * 8);
  h->o_isf = take(nP * 4);
  h->o_tok = take(T * 4);
  h->o_dcnt = take(TP * 4);
  h->o_dmax = take(TP * 4);
  h->o_flt = take((size_t)T * h->nF * 8);
  h->meta_bytes = mo;
  auto dmalloc = [&](size_t bytes) -> void* {
    void* p = atc_pool_alloc(ctx, std::max(bytes, (size_t)256));
    if (p) h->allocations.push_back(p);
    return p;
  };
  double* init = (double*)dmalloc(total * 8);
  double* fin = (double*)dmalloc(total * 8);
  int32_t* dpos = (int32_t*)dmalloc(dtotal * 4);
  h->meta = (uint8_t*)dmalloc(mo);
  if (!init || !fin || !dpos || !h->meta) {
    atc_set_error(ctx, "cudaMalloc failed for %lld region doubles", (long long)total);
    atc_testsets_free(ctx, h);
    return ATC_ERR_CUDA;
  }
  TestsetView& v = h->view;
  v.T = T;
  v.nI = nI;
  v.nP = nP;
  {  // div_nI constants: m = ceil(2^(31 + s) / nI), s = ceil(log2 nI) (exact for n < 2^31)
    uint32_t sh = 0;
    while ((1ull << sh) < (uint64_t)nI) ++sh;
    v.nI_m = nI <= 1 ? 0u : (uint32_t)(((1ull << (31 + sh)) + nI - 1) / (uint64_t)nI);
    v.nI_sh = sh ? sh - 1 : 0;
  }
  v.ints = (const int64_t*)(h->meta + h->o_ints);
  v.is_f32 = (const int32_t*)(h->meta + h->o_isf);
  v.region_len = (const int64_t*)(h->meta + h->o_rlen);
  v.test_ok = (const int32_t*)(h->meta + h->o_tok);
  v.init = init;
  v.fin = fin;
  v.region_off = (const int64_t*)(h->meta + h->o_roff);
  v.dirty_pos = dpos;
  v.dirty_off = (const int64_t*)(h->meta + h->o_dof);
  v.dirty_cnt = (const int32_t*)(h->meta + h->o_dcnt);
  v.dirty_max = (const int32_t*)(h->meta + h->o_dmax);
  v.nF = h->nF;
  v.floats = h->nF ? (const double*)(h->meta + h->o_flt) : nullptr;
  h->cs = ctx->copy_next;  // round-robin over the copy streams
  ctx->copy_next = (h->cs + 1) % atc_ctx::kCopyStreams;
  const int rc = testsets_fill(ctx, h, ts_full, sd, sync, false, nullptr, pre);
  if (rc) {
    atc_testsets_free(ctx, h);
    return rc;
  }
  *out = h;
  return ATC_OK;
}

extern "C" {

int atc_testsets_upload(atc_ctx* ctx, const atc_testsets* ts, atc_testset_handle** out) {
  return testsets_upload(ctx, ts, nullptr, out, true);
}

int atc_testsets_upload_async(atc_ctx* ctx, const atc_testsets* ts, atc_testset_handle** out) {
  return testsets_upload(ctx, ts, nullptr, out, false);
}

int atc_testsets_upload_seeded(atc_ctx* ctx, const atc_seeded_testsets* ts, atc_testset_handle** out) {
  return testsets_upload(ctx, nullptr, ts, out, false);
}

int atc_testsets_upload_prefix(atc_ctx* ctx, const atc_prefix_testsets* ts, atc_testset_handle** out) {
  ATC_ENTER(ctx);
  if (!ts || !ts->init || !ts->diff_off || ts->n_tests < 1 || ts->n_ptrs < 1 || ts->n_tests > kMaxT ||
      ts->n_ptrs > kMaxPtrs) {
    atc_set_error(ctx, "malformed test sets");
    return ATC_ERR_ARG;
  }
  const size_t TP = (size_t)ts->n_tests * ts->n_ptrs;
  for (size_t i = 0; i < TP; ++i)
    if (!ts->init[i] && (!ts->test_ok || ts->test_ok[i / ts->n_ptrs])) {
      atc_set_error(ctx, "test %d pointer %d: missing region", (int)(i / ts->n_ptrs), (int)(i % ts->n_ptrs));
      return ATC_ERR_ARG;
    }
  // the seeded form's header with unused stream fields: the prefixes replace the generator
  std::vector<uint64_t> zeros(TP, 0);
  atc_seeded_testsets sd{ts->n_tests, ts->n_ints,   ts->n_ptrs,   ts->int_values, ts->ptr_is_f32,
                         ts->region_len, ts->test_ok, zeros.data(), zeros.data(),  ts->diff_off,
                         ts->diff_pos,   ts->diff_val, /*needed_only=*/1};
  return testsets_upload(ctx, nullptr, &sd, out, false, ts->init);
}

static bool update_matches(atc_ctx* ctx, const atc_testset_handle* h, const atc_seeded_testsets* ts) {
  if (!h || !ts || ts->n_tests != h->T || ts->n_ints != h->nI || ts->n_ptrs != h->nP || !ts->int_values ||
      !ts->region_len || !ts->ptr_is_f32 || !ts->stream_seed || !ts->stream_skip || !ts->diff_off ||
      ts->diff_off[0] != 0) {
    atc_set_error(ctx, "atc_testsets_update_seeded: test sets do not match the handle");
    return false;
  }
  for (int p = 0; p < h->nP; ++p)
    if (ts->region_len[p] != h->lens[p] || (ts->ptr_is_f32[p] != 0) != (h->is_f32[p] != 0)) {
      atc_set_error(ctx, "atc_testsets_update_seeded: pointer %d differs from the handle's", p);
      return false;
    }
  return true;
}

int atc_testsets_update_seeded(atc_ctx* ctx, atc_testset_handle* h, const atc_seeded_testsets* ts) {
  return atc_testsets_update_seeded_many(ctx, &h, ts, 1);
}

// Batched in-place update of distinct needed_only handles (the prepared-sweep step's
// call), in groups of kUpdGroup handles in call order.  Each group's metadata blocks,
// seeds, stream positions, final-minus-init entries and prefix bounds are packed into
// its own slice of one pinned staging buffer; as soon as a slice is packed it goes out
// as one H2D and one k_copy_meta on copy stream 0 and the group's generators as one
// k_probe_regions_many launch on copy stream 1, 2, ..., each handle's ready event after
// it — so the first generators start while the host still packs the later groups
// (packing everything before the first copy held the GPU idle for ~0.13 ms), and per
// handle two copies, a launch and an event from four host threads are gone.  Callers
// list the handles whose evaluations start the longest chains first.
static int update_seeded_batched(atc_ctx* ctx, atc_testset_handle* const* handles, const atc_seeded_testsets* ts,
                                 int32_t n) {
  constexpr int kUpdGroup = 4;
  struct Lay {
    size_t meta, seeds, skips, doffs, dvs, dps, need;
  };
  const int n_groups = (n + kUpdGroup - 1) / kUpdGroup;
  std::vector<Lay> lay((size_t)n);
  std::vector<size_t> g_off((size_t)n_groups + 1);
  size_t bytes = 0;
  auto take = [&](size_t b) {
    const size_t o = bytes;
    bytes += (b + 15) / 16 * 16;
    return o;
  };
  for (int i = 0; i < n; ++i) {
    if (i % kUpdGroup == 0) {  // a group's slice starts with its jobs
      bytes = (bytes + 255) / 256 * 256;
      g_off[(size_t)(i / kUpdGroup)] = bytes;
      take((size_t)kUpdGroup * sizeof(atc::ProbeJob));
    }
    const atc_testset_handle* h = handles[i];
    const size_t TP = (size_t)h->T * h->nP;
    const int64_t nd = ts[i].diff_off[TP];
    for (int64_t e = 0; e < nd; ++e)
      if (ts[i].diff_pos[e] < 0) {
        atc_set_error(ctx, "negative final-minus-init position");
        return ATC_ERR_ARG;
      }
    lay[i] = {take(h->meta_bytes), take((size_t)h->T * 8), take(TP * 8), take((TP + 1) * 8), take((size_t)nd * 8),
              take((size_t)nd * 4), take(TP * 8)};
  }
  g_off[(size_t)n_groups] = bytes;
  // the staging of the previous batched update must have been copied out
  if (ctx->upd_h2d_ev && !atc_cuda_ok(ctx, cudaEventSynchronize(ctx->upd_h2d_ev), "update staging reuse"))
    return ATC_ERR_CUDA;
  if (ctx->upd_cap < bytes) {
    if (ctx->upd_pin) cudaFreeHost(ctx->upd_pin);
    if (ctx->upd_dev) cudaFree(ctx->upd_dev);
    ctx->upd_pin = nullptr;
    ctx->upd_dev = nullptr;
    ctx->upd_cap = 0;
    if (!atc_cuda_ok(ctx, cudaMallocHost(&ctx->upd_pin, bytes), "cudaMallocHost") ||
        !atc_cuda_ok(ctx, cudaMalloc(&ctx->upd_dev, bytes), "cudaMalloc"))
      return ATC_ERR_CUDA;
    ctx->upd_cap = bytes;
  }
  if (!ctx->upd_h2d_ev) {
    bool ok = atc_cuda_ok(ctx, cudaEventCreateWithFlags(&ctx->upd_h2d_ev, cudaEventDisableTiming), "cudaEventCreate") &&
              atc_cuda_ok(ctx, cudaEventCreateWithFlags(&ctx->upd_meta_ev, cudaEventDisableTiming), "cudaEventCreate");
    for (int k = 0; k < atc_ctx::kCopyStreams && ok; ++k)
      ok = atc_cuda_ok(ctx, cudaEventCreateWithFlags(&ctx->upd_done_ev[k], cudaEventDisableTiming), "cudaEventCreate");
    if (!ok) return ATC_ERR_CUDA;
  }
  uint8_t* hp = ctx->upd_pin;
  uint8_t* dp = ctx->upd_dev;
  cudaStream_t st = ctx->copy_stream[0];
  if (ctx->free_pending & 1ull) {
    cudaStreamWaitEvent(st, ctx->free_ev, 0);
    ctx->free_pending &= ~1ull;
  }
  cudaStreamWaitEvent(st, ctx->update_ev, 0);  // earlier readers of the old contents first
  for (int i = 0; i < n; ++i)                   // and every handle's earlier uploads
    if (handles[i]->ready) cudaStreamWaitEvent(st, handles[i]->ready, 0);
  bool ok = true;
  for (int g = 0; g < n_groups && ok; ++g) {
    const int i0 = g * kUpdGroup, i1 = std::min(n, i0 + kUpdGroup);
    auto* jobs = reinterpret_cast<atc::ProbeJob*>(hp + g_off[(size_t)g]);
    int g_ctas = 0;
    for (int i = i0; i < i1; ++i) {
      atc_testset_handle* h = handles[i];
      const atc_seeded_testsets& sd = ts[i];
      const size_t TP = (size_t)h->T * h->nP;
      const int64_t nd = sd.diff_off[TP];
      const Lay& L = lay[i];
      h->h_ints.assign(sd.int_values, sd.int_values + (size_t)h->T * h->nI);
      h->needed_only = true;
      fill_meta(h, sd.int_values, sd.test_ok, nullptr, hp + L.meta);
      std::memcpy(hp + L.seeds, sd.stream_seed, (size_t)h->T * 8);
      std::memcpy(hp + L.skips, sd.stream_skip, TP * 8);
      std::memcpy(hp + L.doffs, sd.diff_off, (TP + 1) * 8);
      if (nd) {
        std::memcpy(hp + L.dvs, sd.diff_val, (size_t)nd * 8);
        std::memcpy(hp + L.dps, sd.diff_pos, (size_t)nd * 4);
      }
      const std::vector<int64_t> need = region_need(h, &sd);
      std::memcpy(hp + L.need, need.data(), TP * 8);
      atc::ProbeJob& b = jobs[i - i0];
      b.view = h->view;
      b.cta0 = g_ctas;  // CTA numbering restarts per launch group
      g_ctas += h->T;
      b.seeds = (const uint64_t*)(dp + L.seeds);
      b.skips = (const uint64_t*)(dp + L.skips);
      b.diff_off = (const int64_t*)(dp + L.doffs);
      b.diff_pos = (const int32_t*)(dp + L.dps);
      b.diff_val = (const double*)(dp + L.dvs);
      b.need = (const int64_t*)(dp + L.need);
      b.meta_src = dp + L.meta;
      b.meta_dst = h->meta;
      b.meta_bytes = h->meta_bytes;
    }
    const size_t o = g_off[(size_t)g], len = g_off[(size_t)g + 1] - o;
    const atc::ProbeJob* dj = reinterpret_cast<const atc::ProbeJob*>(dp + o);
    ok = atc_cuda_ok(ctx, cudaMemcpyAsync(dp + o, hp + o, len, cudaMemcpyHostToDevice, st), "H2D update batch");
    if (!ok) break;
    atc::k_copy_meta<<<(unsigned)(i1 - i0), 256, 0, st>>>(dj);
    ok = atc_cuda_ok(ctx, cudaGetLastError(), "k_copy_meta") &&
         atc_cuda_ok(ctx, cudaEventRecord(ctx->upd_meta_ev, st), "cudaEventRecord");
    if (!ok) break;
    cudaStream_t gs = ctx->copy_stream[1 + g % (atc_ctx::kCopyStreams - 1)];
    cudaStreamWaitEvent(gs, ctx->upd_meta_ev, 0);
    atc::k_probe_regions_many<<<(unsigned)g_ctas, atc::kProbeThreads, 0, gs>>>(dj, i1 - i0);
    ok = atc_cuda_ok(ctx, cudaGetLastError(), "k_probe_regions_many");
    for (int i = i0; i < i1 && ok; ++i) {
      atc_testset_handle* h = handles[i];
      ok = (h->ready || atc_cuda_ok(ctx, cudaEventCreateWithFlags(&h->ready, cudaEventDisableTiming), "cudaEventCreate")) &&
           atc_cuda_ok(ctx, cudaEventRecord(h->ready, gs), "cudaEventRecord");
    }
    ok = ok && atc_cuda_ok(ctx, cudaEventRecord(ctx->upd_done_ev[g % atc_ctx::kCopyStreams], gs), "cudaEventRecord");
  }
  ok = ok && atc_cuda_ok(ctx, cudaEventRecord(ctx->upd_h2d_ev, st), "cudaEventRecord");
  // the next batch's staging copies (stream 0) after every generator has read this one
  for (int g = 0; g < n_groups && ok; ++g) cudaStreamWaitEvent(st, ctx->upd_done_ev[g % atc_ctx::kCopyStreams], 0);
  return ok ? ATC_OK : ATC_ERR_CUDA;
}

int atc_testsets_update_seeded_many(atc_ctx* ctx, atc_testset_handle* const* handles, const atc_seeded_testsets* ts,
                                    int32_t n) {
  ATC_ENTER(ctx);
  if (n < 0 || (n > 0 && (!handles || !ts))) {
    atc_set_error(ctx, "bad arguments to atc_testsets_update_seeded_many");
    return ATC_ERR_ARG;
  }
  for (int i = 0; i < n; ++i)
    if (!update_matches(ctx, handles[i], ts + i)) return ATC_ERR_ARG;
  if (n == 0) return ATC_OK;
  cudaSetDevice(ctx->device);
  // the new contents are written after everything queued so far on the compute
  // stream (evaluations of every sweep branch join it) has read the old ones: one
  // event for the whole set of updates
  if (!ctx->update_ev &&
      !atc_cuda_ok(ctx, cudaEventCreateWithFlags(&ctx->update_ev, cudaEventDisableTiming), "cudaEventCreate"))
    return ATC_ERR_CUDA;
  if (!atc_cuda_ok(ctx, cudaEventRecord(ctx->update_ev, ctx->stream), "cudaEventRecord")) return ATC_ERR_CUDA;
  // shared context state first, serially: pool growth of the seeded blocks and the
  // copy streams' waits on earlier frees; then the per-handle work (staging, H2D,
  // generator launch) on up to four host threads when the handles are distinct
  bool distinct = true;
  for (int i = 0; i < n && distinct; ++i) {
    atc_testset_handle* h = handles[i];
    for (int k = 0; k < i; ++k) distinct = distinct && handles[k] != h;
    const size_t TP = (size_t)h->T * h->nP;
    const int64_t nd = ts[i].diff_off[TP];
    const size_t so = ((size_t)h->T * 8 + 15) / 16 * 16 + (TP * 8 + 15) / 16 * 16 + ((TP + 1) * 8 + 15) / 16 * 16 +
                      ((size_t)nd * 8 + 15) / 16 * 16 + ((size_t)nd * 4 + 15) / 16 * 16 + (TP * 8 + 15) / 16 * 16;
    if (so > h->seeded_cap) {
      h->seeded = (uint8_t*)atc_pool_alloc(ctx, std::max(so, (size_t)256));
      if (!h->seeded) {
        h->seeded_cap = 0;
        atc_set_error(ctx, "device allocation failed (seeded test sets)");
        return ATC_ERR_CUDA;
      }
      h->allocations.push_back(h->seeded);
      h->seeded_cap = so;
    }
    if (ctx->free_pending & (1ull << h->cs)) {
      cudaStreamWaitEvent(ctx->copy_stream[h->cs], ctx->free_ev, 0);
      ctx->free_pending &= ~(1ull << h->cs);
    }
  }
  if (distinct && n > 1) {
    bool batchable = true;
    for (int i = 0; i < n && batchable; ++i) batchable = ts[i].needed_only != 0;
    if (batchable) return update_seeded_batched(ctx, handles, ts, n);
  }
  const int workers = distinct ? std::min(n, 4) : 1;
  std::atomic<int> first_rc{ATC_OK};
  auto work = [&](int w) {
    cudaSetDevice(ctx->device);
    for (int i = w; i < n; i += workers) {
      const int rc = testsets_fill(ctx, handles[i], nullptr, ts + i, false, true, ctx->update_ev);
      if (rc) {
        int expected = ATC_OK;
        first_rc.compare_exchange_strong(expected, rc);
        return;
      }
    }
  };
  std::vector<std::thread> pool;
  for (int w = 1; w < workers; ++w) pool.emplace_back(work, w);
  work(0);
  for (auto& th : pool) th.join();
  return first_rc.load();
}

int atc_testsets_download(atc_ctx* ctx, const atc_testset_handle* h, double* init, double* final_) {
  ATC_ENTER(ctx);
  if (!h || (!init && !final_)) {
    atc_set_error(ctx, "bad arguments to atc_testsets_download");
    return ATC_ERR_ARG;
  }
  if (h->needed_only) {
    atc_set_error(ctx, "atc_testsets_download: the handle holds only the needed region prefixes");
    return ATC_ERR_ARG;
  }
  cudaSetDevice(ctx->device);
  if (h->ready && !atc_cuda_ok(ctx, cudaEventSynchronize(h->ready), "upload wait")) return ATC_ERR_CUDA;
  std::vector<int64_t> off((size_t)h->T * h->nP), len(h->nP);
  if (!atc_cuda_ok(ctx, cudaMemcpy(off.data(), h->view.region_off, off.size() * 8, cudaMemcpyDeviceToHost), "D2H") ||
      !atc_cuda_ok(ctx, cudaMemcpy(len.data(), h->view.region_len, len.size() * 8, cudaMemcpyDeviceToHost), "D2H"))
    return ATC_ERR_CUDA;
  size_t o = 0;  // host layout: (t, p) regions back to back, unpadded
  for (int t = 0; t < h->T; ++t)
    for (int p = 0; p < h->nP; ++p) {
      const size_t i = (size_t)t * h->nP + p, bytes = (size_t)len[p] * 8;
      if ((init && !atc_cuda_ok(ctx, cudaMemcpy(init + o, h->view.init + off[i], bytes, cudaMemcpyDeviceToHost), "D2H")) ||
          (final_ && !atc_cuda_ok(ctx, cudaMemcpy(final_ + o, h->view.fin + off[i], bytes, cudaMemcpyDeviceToHost), "D2H")))
        return ATC_ERR_CUDA;
      o += (size_t)len[p];
    }
  return ATC_OK;
}

int atc_testsets_free(atc_ctx* ctx, atc_testset_handle* h) {
  if (!h) return ATC_OK;
  AtcLock lock(ctx);
  if (ctx && !ctx->broken) {
    cudaSetDevice(ctx->device);
    // the memory returns to the pool: later uploads wait until the compute
    // stream has passed this point (and this handle's own copies are done)
    ts_wait(h, ctx->stream);
    cudaEventRecord(ctx->free_ev, ctx->stream);
    ctx->free_pending = (atc_ctx::kCopyStreams >= 64) ? ~0ull : (1ull << atc_ctx::kCopyStreams) - 1;
  }
  if (h->ready) {
    cudaEventSynchronize(h->ready);  // the staging buffer may still be read by its DMA
    cudaEventDestroy(h->ready);
  }
  if (h->pin) cudaFreeHost(h->pin);
  for (void* p : h->allocations) {
    if (ctx && !ctx->broken)
      atc_pool_free(ctx, p);
    else
      cudaFree(p);
  }
  delete h;
  return ATC_OK;
}

}  // extern "C"
