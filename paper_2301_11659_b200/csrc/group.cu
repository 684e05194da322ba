// C ABI: device groups — one context per GPU of one process,
// enumerated ranges sharded over them, results combined on the host.
//
// The reference evaluates candidates one at a time inside lift_function
// (pipeline.cpp:248-310), one function per worker thread (pipeline.cpp:340-355).
// Here a range of the unpruned space (Appendix C order) is cut into contiguous
// pieces by the shard plan; each device evaluates its pieces against its own
// replica of the recorded test sets (no data-path exchange) and returns its
// result block; the group combines them: MIN of the first passing index (the
// candidate a rank-order loop reaches first), SUM of the reason histograms, the
// ordered union of the passing lists.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "atc_b200.h"
#include "capi_internal.h"

namespace {

// Cost model of one piece of a large (conv) space on one B200 (tools/rank_breakdown.py,
// r2 kernels): a fixed part (position tables, K2, finalize) plus the K1 screen per
// binding.  workloads.py carries the same constants.
constexpr uint64_t kBigSpace = 1ull << 24;
constexpr double kSpaceFixedMs = 0.10;
const double kSpaceMsPerBinding = 0.123 / 2324522934.0;

double space_cost_ms(uint64_t n) { return n > 0 ? kSpaceFixedMs + (double)n * kSpaceMsPerBinding : 0.0; }

uint64_t block_edge(uint64_t n, uint64_t idx, uint64_t k) {
  return (uint64_t)((unsigned __int128)n * idx / k);
}

// begin/end [world][n]: see atc_plan_shards in include/atc_b200.h
void plan(const uint64_t* counts, int n, int world, uint64_t* begin, uint64_t* end) {
  for (int i = 0; i < world * n; ++i) begin[i] = end[i] = 0;
  if (world == 1) {
    for (int j = 0; j < n; ++j) end[j] = counts[j];
    return;
  }
  std::vector<int> big;
  for (int j = 0; j < n; ++j)
    if (counts[j] >= kBigSpace) big.push_back(j);
  double target = 0.0;
  for (int j : big) target += space_cost_ms(counts[j]);
  target /= world;
  std::vector<double> load(world, 0.0);
  std::sort(big.begin(), big.end(), [&](int a, int b) {
    return counts[a] != counts[b] ? counts[a] > counts[b] : a < b;
  });
  std::vector<char> is_big(n, 0);
  for (int j : big) {
    is_big[j] = 1;
    const uint64_t c = counts[j];
    std::vector<int> order(world);
    for (int r = 0; r < world; ++r) order[r] = r;
    std::sort(order.begin(), order.end(), [&](int a, int b) { return load[a] != load[b] ? load[a] < load[b] : a < b; });
    // the fewest pieces that keep every receiving rank within the target (+15%),
    // else the piece count with the lowest resulting maximum
    int fits = 0, best_k = 0;
    double best = 0.0;
    for (int k = 1; k <= world; ++k) {
      const double peak = load[order[k - 1]] + space_cost_ms((c + k - 1) / k);
      if (!fits && peak <= 1.15 * target) fits = k;
      if (!best_k || peak < best - 1e-12) {
        best = peak;
        best_k = k;
      }
    }
    const int k = fits ? fits : best_k;
    std::vector<int> ranks(order.begin(), order.begin() + k);
    std::sort(ranks.begin(), ranks.end());
    for (int idx = 0; idx < k; ++idx) {
      const int r = ranks[idx];
      begin[(size_t)r * n + j] = block_edge(c, idx, k);
      end[(size_t)r * n + j] = block_edge(c, idx + 1, k);
      load[r] += space_cost_ms(end[(size_t)r * n + j] - begin[(size_t)r * n + j]);
    }
  }
  int dealt = 0;
  for (int j = 0; j < n; ++j) {
    if (is_big[j]) continue;
    const int r = dealt++ % world;
    end[(size_t)r * n + j] = counts[j];
  }
}

}  // namespace

struct atc_group {
  std::vector<atc_ctx*> members;
  std::string err;
  std::recursive_mutex mu;
};

struct atc_group_testsets {
  std::vector<atc_testset_handle*> h;  // one per member
};

// One member's share of a group sweep: its enumerated jobs (non-empty pieces only),
// the group job each maps to, and a survivor buffer per piece.
struct MemberShare {
  std::vector<atc_enum_job> jobs;
  std::vector<int> of;
  std::vector<std::vector<uint64_t>> bufs;
};

struct atc_group_batch {
  atc_group_job* jobs = nullptr;
  int n = 0;
  std::vector<MemberShare> shares;
  std::vector<atc_enum_batch*> batches;  // per member (nullptr: no share)
};

namespace {

void group_error(atc_group* g, const std::string& msg) { g->err = msg; }

// The shares of every member; returns false (with the group error) on bad jobs.
bool make_shares(atc_group* g, atc_group_job* jobs, int n_jobs, std::vector<MemberShare>& shares) {
  const int world = (int)g->members.size();
  std::vector<uint64_t> counts(n_jobs), b((size_t)world * n_jobs), e((size_t)world * n_jobs);
  for (int j = 0; j < n_jobs; ++j) {
    atc_group_job& jb = jobs[j];
    jb.status = ATC_OK;
    jb.n_survivors = 0;
    jb.first_pass = -1;
    for (auto& r : jb.reason_counts) r = 0;
    if (!jb.ts || (int)jb.ts->h.size() != world || jb.end < jb.begin || jb.cap < 0) {
      group_error(g, "bad arguments to atc_group_eval_enumerated_many (job " + std::to_string(j) + ")");
      return false;
    }
    counts[j] = jb.end - jb.begin;
  }
  plan(counts.data(), n_jobs, world, b.data(), e.data());
  shares.assign(world, MemberShare{});
  for (int m = 0; m < world; ++m) {
    MemberShare& s = shares[m];
    for (int j = 0; j < n_jobs; ++j) {
      const uint64_t lo = b[(size_t)m * n_jobs + j], hi = e[(size_t)m * n_jobs + j];
      if (hi <= lo) continue;
      const atc_group_job& jb = jobs[j];
      atc_enum_job ej{};
      ej.spec = jb.spec;
      ej.ts = jb.ts->h[m];
      ej.perms = jb.perms;
      ej.n_perms = jb.n_perms;
      ej.begin = jb.begin + lo;
      ej.end = jb.begin + hi;
      ej.cap = std::max<int64_t>(jb.cap, 1);  // at least the first passing index
      s.jobs.push_back(ej);
      s.of.push_back(j);
      s.bufs.emplace_back((size_t)ej.cap);
    }
    for (size_t i = 0; i < s.jobs.size(); ++i) s.jobs[i].survivors = s.bufs[i].data();
  }
  return true;
}

// Runs fn(m) for every member, concurrently (one host thread per member).
template <class F>
void for_members(int world, F fn) {
  if (world == 1) {
    fn(0);
    return;
  }
  std::vector<std::thread> th;
  for (int m = 1; m < world; ++m) th.emplace_back(fn, m);
  fn(0);
  for (auto& t : th) t.join();
}

// The combine step: per group job, MIN / SUM / ordered union over the members.
int combine(atc_group* g, atc_group_job* jobs, int n_jobs, const std::vector<MemberShare>& shares,
            const std::vector<int>& rc) {
  std::vector<std::vector<uint64_t>> pass(n_jobs);
  int first_rc = ATC_OK;
  for (size_t m = 0; m < shares.size(); ++m) {
    const MemberShare& s = shares[m];
    for (size_t i = 0; i < s.jobs.size(); ++i) {
      const atc_enum_job& ej = s.jobs[i];
      atc_group_job& jb = jobs[s.of[i]];
      const int st = ej.status != ATC_OK ? ej.status : rc[m];
      if (st != ATC_OK) {
        if (jb.status == ATC_OK) jb.status = st;
        if (first_rc == ATC_OK) {
          first_rc = st;
          group_error(g, "device " + std::to_string(g->members[m]->device) + ": " + g->members[m]->err);
        }
        continue;
      }
      jb.n_survivors += ej.n_survivors;
      for (int r = 0; r < ATC_REASON_COUNT; ++r) jb.reason_counts[r] += ej.reason_counts[r];
      const int64_t have = std::min<int64_t>(ej.n_survivors, ej.cap);
      pass[s.of[i]].insert(pass[s.of[i]].end(), s.bufs[i].begin(), s.bufs[i].begin() + have);
    }
  }
  for (int j = 0; j < n_jobs; ++j) {
    atc_group_job& jb = jobs[j];
    std::sort(pass[j].begin(), pass[j].end());
    jb.first_pass = pass[j].empty() ? -1 : (int64_t)pass[j][0];
    for (size_t i = 0; i < pass[j].size() && (int64_t)i < jb.cap; ++i)
      if (jb.survivors) jb.survivors[i] = pass[j][i];
  }
  return first_rc;
}

int group_ok(atc_group* g) {
  if (!g || g->members.empty()) return ATC_ERR_ARG;
  for (atc_ctx* c : g->members)
    if (c->broken) return ATC_ERR_DEVICE;
  return ATC_OK;
}

template <class Up>
int group_upload(atc_group* g, atc_group_testsets** out, Up up) {
  if (int rc = group_ok(g)) return rc;
  std::lock_guard<std::recursive_mutex> lk(g->mu);
  if (!out) return ATC_ERR_ARG;
  auto* h = new atc_group_testsets();
  for (atc_ctx* c : g->members) {
    atc_testset_handle* m = nullptr;
    if (int rc = up(c, &m)) {
      group_error(g, "device " + std::to_string(c->device) + ": " + c->err);
      atc_group_testsets_free(g, h);
      return rc;
    }
    h->h.push_back(m);
  }
  *out = h;
  return ATC_OK;
}

}  // namespace

extern "C" {

int atc_plan_shards(const uint64_t* counts, int32_t n_jobs, int32_t world, uint64_t* begin, uint64_t* end) {
  if (n_jobs < 0 || world < 1 || (n_jobs > 0 && (!counts || !begin || !end))) return ATC_ERR_ARG;
  plan(counts, n_jobs, world, begin, end);
  return ATC_OK;
}

atc_group* atc_group_create(const int32_t* devices, int32_t n) {
  auto* g = new atc_group();
  if (n <= 0) {
    n = atc_device_count();
    devices = nullptr;
  }
  if (n <= 0) {
    group_error(g, "no CUDA device");
    return g;
  }
  for (int i = 0; i < n; ++i) {
    atc_ctx* c = atc_create(devices ? devices[i] : i);
    g->members.push_back(c);
    if (c->broken && g->err.empty()) group_error(g, "device " + std::to_string(c->device) + ": " + c->err);
  }
  // peer access between distinct member devices (NVLink / NVSwitch), for callers that
  // move data between members' buffers; not needed by the combine itself
  for (atc_ctx* a : g->members)
    for (atc_ctx* b : g->members) {
      int can = 0;
      if (a->broken || b->broken || a->device == b->device) continue;
      if (cudaDeviceCanAccessPeer(&can, a->device, b->device) == cudaSuccess && can) {
        cudaSetDevice(a->device);
        if (cudaDeviceEnablePeerAccess(b->device, 0) != cudaSuccess) cudaGetLastError();  // already enabled
      }
    }
  return g;
}

void atc_group_destroy(atc_group* g) {
  if (!g) return;
  for (atc_ctx* c : g->members) atc_destroy(c);
  delete g;
}

const char* atc_group_last_error(const atc_group* g) { return g ? g->err.c_str() : "null group"; }

int32_t atc_group_size(const atc_group* g) { return g ? (int32_t)g->members.size() : 0; }

atc_ctx* atc_group_member(atc_group* g, int32_t i) {
  return g && i >= 0 && i < (int32_t)g->members.size() ? g->members[i] : nullptr;
}

int atc_group_testsets_upload_seeded(atc_group* g, const atc_seeded_testsets* ts, atc_group_testsets** out) {
  return group_upload(g, out, [&](atc_ctx* c, atc_testset_handle** m) { return atc_testsets_upload_seeded(c, ts, m); });
}

int atc_group_testsets_upload_prefix(atc_group* g, const atc_prefix_testsets* ts, atc_group_testsets** out) {
  return group_upload(g, out, [&](atc_ctx* c, atc_testset_handle** m) { return atc_testsets_upload_prefix(c, ts, m); });
}

int atc_group_testsets_free(atc_group* g, atc_group_testsets* h) {
  if (!h) return ATC_OK;
  for (size_t i = 0; i < h->h.size(); ++i)
    atc_testsets_free(g && i < g->members.size() ? g->members[i] : nullptr, h->h[i]);
  delete h;
  return ATC_OK;
}

const atc_testset_handle* atc_group_testsets_member(const atc_group_testsets* h, int32_t i) {
  return h && i >= 0 && i < (int32_t)h->h.size() ? h->h[i] : nullptr;
}

int atc_group_eval_enumerated_many(atc_group* g, atc_group_job* jobs, int32_t n_jobs, int32_t mode) {
  if (int rc = group_ok(g)) return rc;
  std::lock_guard<std::recursive_mutex> lk(g->mu);
  if (n_jobs < 0 || (n_jobs > 0 && !jobs)) return ATC_ERR_ARG;
  std::vector<MemberShare> shares;
  if (!make_shares(g, jobs, n_jobs, shares)) return ATC_ERR_ARG;
  std::vector<int> rc(g->members.size(), ATC_OK);
  for_members((int)g->members.size(), [&](int m) {
    MemberShare& s = shares[m];
    if (!s.jobs.empty()) rc[m] = atc_eval_enumerated_many(g->members[m], s.jobs.data(), (int32_t)s.jobs.size(), mode);
  });
  return combine(g, jobs, n_jobs, shares, rc);
}

atc_group_batch* atc_group_batch_create(atc_group* g, atc_group_job* jobs, int32_t n_jobs, int32_t mode) {
  if (group_ok(g) != ATC_OK || n_jobs < 0 || (n_jobs > 0 && !jobs)) {
    if (g) group_error(g, "bad arguments to atc_group_batch_create");
    return nullptr;
  }
  std::lock_guard<std::recursive_mutex> lk(g->mu);
  auto* b = new atc_group_batch();
  b->jobs = jobs;
  b->n = n_jobs;
  if (!make_shares(g, jobs, n_jobs, b->shares)) {
    delete b;
    return nullptr;
  }
  b->batches.assign(g->members.size(), nullptr);
  bool ok = true;
  for (size_t m = 0; m < g->members.size(); ++m) {
    MemberShare& s = b->shares[m];
    if (s.jobs.empty()) continue;
    b->batches[m] = atc_enum_batch_create(g->members[m], s.jobs.data(), (int32_t)s.jobs.size(), mode);
    if (!b->batches[m]) {
      group_error(g, "device " + std::to_string(g->members[m]->device) + ": " + g->members[m]->err);
      ok = false;
      break;
    }
  }
  if (!ok) {
    atc_group_batch_destroy(g, b);
    return nullptr;
  }
  return b;
}

int atc_group_batch_run(atc_group* g, atc_group_batch* b) {
  if (int rc = group_ok(g)) return rc;
  if (!b) return ATC_ERR_ARG;
  std::lock_guard<std::recursive_mutex> lk(g->mu);
  for (int j = 0; j < b->n; ++j) {
    atc_group_job& jb = b->jobs[j];
    jb.status = ATC_OK;
    jb.n_survivors = 0;
    jb.first_pass = -1;
    for (auto& r : jb.reason_counts) r = 0;
  }
  std::vector<int> rc(g->members.size(), ATC_OK);
  for_members((int)g->members.size(), [&](int m) {
    if (b->batches[m]) rc[m] = atc_enum_batch_run(g->members[m], b->batches[m]);
  });
  return combine(g, b->jobs, b->n, b->shares, rc);
}

void atc_group_batch_destroy(atc_group* g, atc_group_batch* b) {
  if (!b) return;
  for (size_t m = 0; m < b->batches.size(); ++m)
    if (b->batches[m]) atc_enum_batch_destroy(g ? g->members[m] : nullptr, b->batches[m]);
  delete b;
}

}  // extern "C"
