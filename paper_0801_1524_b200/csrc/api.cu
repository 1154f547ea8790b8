// api.cu -- the C ABI of include/sft.h: plan / apply / destroy and the
// multi-GPU phase calls.  Host orchestration only; every arithmetic step of
// the transform runs in the kernels of tree.cu and kernels.cu.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "sft_internal.cuh"

using namespace sft;

static thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CKR(x)                                                                   \
  do {                                                                           \
    cudaError_t e_ = (x);                                                        \
    if (e_ != cudaSuccess)                                                       \
      return fail(SFT_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));  \
  } while (0)

// one non-blocking side stream per device for the plan's schedule kernel
static cudaStream_t side_stream() {
  static cudaStream_t st[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!st[dev]) cudaStreamCreateWithFlags(&st[dev], cudaStreamNonBlocking);
  return st[dev];
}

static bool is_device_ptr(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();  // clear
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

static int64_t ipow64(int b, int e) {
  int64_t r = 1;
  while (e-- > 0) r *= b;
  return r;
}

extern "C" void sft_default_opts(sft_opts* o) {
  if (!o) return;
  o->precision = 0;
  o->stream = nullptr;
  o->rank = 0;
  o->world = 1;
  o->exchange_level = -1;
  o->split_k = -1;
  o->split_x = -1;
  o->adjoint = 0;
  o->nccl_id = nullptr;
}

extern "C" const char* sft_strerror(int status) {
  switch (status) {
    case SFT_OK: return "ok";
    case SFT_E_ARG: return "invalid argument";
    case SFT_E_DOMAIN: return "coordinate outside [0,N] or non-finite";
    case SFT_E_NOMEM: return "out of memory";
    case SFT_E_CUDA: return "CUDA error";
    case SFT_E_STATE: return "invalid call for this plan";
    case SFT_E_NCCL: return "NCCL error";
    default: return "unknown status";
  }
}

extern "C" const char* sft_last_error(void) { return g_last_error.c_str(); }

// ---------------------------------------------------------------------------
// ranges of descendants (Morton order keeps every subtree contiguous)
// ---------------------------------------------------------------------------
// For boxes [lo, hi) at level s, the descendant range at level l >= s is
// [first index at l whose ancestor at s is >= lo, ... >= hi).  Computed on the
// host from parent arrays.
static void descend_ranges(const std::vector<std::vector<int32_t>>& parent, int s, int64_t lo, int64_t hi, int L,
                           std::vector<LevelRange>& out) {
  out.assign(L + 1, LevelRange());
  out[s].lo = lo;
  out[s].hi = hi;
  // ancestor-at-s of each box at deeper levels, level by level
  std::vector<int32_t> anc_prev, anc;
  for (int l = s + 1; l <= L; ++l) {
    const std::vector<int32_t>& par = parent[l];
    anc.resize(par.size());
    for (size_t i = 0; i < par.size(); ++i) anc[i] = (l == s + 1) ? par[i] : anc_prev[par[i]];
    out[l].lo = std::lower_bound(anc.begin(), anc.end(), (int32_t)lo) - anc.begin();
    out[l].hi = std::lower_bound(anc.begin(), anc.end(), (int32_t)hi) - anc.begin();
    anc_prev.swap(anc);
  }
  for (int l = 0; l < s; ++l) out[l].lo = out[l].hi = 0;  // unused
}

// ---------------------------------------------------------------------------
// host partitioner; exposed as sft_choose_partition
// ---------------------------------------------------------------------------
// Per-box descendant counts at each level for every box at split level s:
//   cnt[l][i] = number of descendants at level l of box i (level s).
static std::vector<std::vector<int64_t>> desc_counts(const std::vector<std::vector<int32_t>>& parent,
                                                     const std::vector<int64_t>& counts, int s, int L) {
  std::vector<std::vector<int64_t>> cnt(L + 1, std::vector<int64_t>(counts[s], 0));
  std::vector<int32_t> anc_prev, anc;
  for (int64_t i = 0; i < counts[s]; ++i) cnt[s][i] = 1;
  for (int l = s + 1; l <= L; ++l) {
    anc.resize(counts[l]);
    for (int64_t i = 0; i < counts[l]; ++i) {
      anc[i] = (l == s + 1) ? parent[l][i] : anc_prev[parent[l][i]];
      cnt[l][anc[i]]++;
    }
    anc_prev.swap(anc);
  }
  return cnt;
}

// contiguous split of weights w[0..n) into k chunks minimising the max chunk
// (binary search on the bottleneck + greedy), returns boundaries [k+1]
static std::vector<int64_t> linear_partition(const std::vector<int64_t>& w, int k) {
  const int64_t n = (int64_t)w.size();
  int64_t lo = 0, hi = 0;
  for (int64_t v : w) {
    lo = std::max(lo, v);
    hi += v;
  }
  auto feasible = [&](int64_t cap, std::vector<int64_t>* b) {
    int used = 1;
    int64_t cur = 0;
    if (b) {
      b->assign(1, 0);
    }
    for (int64_t i = 0; i < n; ++i) {
      if (cur + w[i] > cap) {
        ++used;
        cur = 0;
        if (b) b->push_back(i);
      }
      cur += w[i];
    }
    return used <= k;
  };
  while (lo < hi) {
    int64_t mid = lo + (hi - lo) / 2;
    if (feasible(mid, nullptr)) hi = mid; else lo = mid + 1;
  }
  std::vector<int64_t> b;
  feasible(lo, &b);
  while ((int)b.size() < k) b.push_back(n);  // empty trailing chunks
  b.push_back(n);
  return b;
}

static int choose_partition(int L, int world, const std::vector<int64_t>& cx, const std::vector<int64_t>& ck,
                            const std::vector<std::vector<int32_t>>& px, const std::vector<std::vector<int32_t>>& pk,
                            int force_sk, int force_sx, int force_m, Partition& best, int64_t* best_cost) {
  int64_t best_total = -1;
  // candidate split levels: forced value, else levels with at least `world`
  // subtrees and few enough (<= 64 per rank) that the search stays cheap;
  // fall back to every level if none qualifies
  auto candidates = [&](const std::vector<int64_t>& c, int force) {
    std::vector<int> v;
    if (force >= 0) {
      if (force <= L) v.push_back(force);
      return v;
    }
    for (int s = 0; s <= L; ++s)
      if (c[s] >= world && c[s] <= 64 * (int64_t)world) v.push_back(s);
    if (v.empty())
      for (int s = 0; s <= L; ++s)
        if (c[s] <= 64 * (int64_t)world) v.push_back(s);
    return v;
  };
  std::vector<int> cand_k = candidates(ck, force_sk), cand_x = candidates(cx, force_sx);
  std::vector<std::vector<std::vector<int64_t>>> DK(L + 1), DX(L + 1);
  for (int s : cand_k) DK[s] = desc_counts(pk, ck, s, L);
  for (int s : cand_x) DX[s] = desc_counts(px, cx, s, L);
  // pairs(t) = ck[t] * cx[L-t]
  for (int sk : cand_k) {
    const auto& dk = DK[sk];
    for (int sx : cand_x) {
      const auto& dx = DX[sx];
      for (int m = sk; m <= L - sx; ++m) {
        if (force_m >= 0 && m != force_m) continue;
        // phase-1 work of T_K box i at sk: sum_{t=m..L} desc_t(i) * cx[L-t]
        std::vector<int64_t> wk(ck[sk], 0), wx(cx[sx], 0);
        for (int64_t i = 0; i < ck[sk]; ++i)
          for (int t = m; t <= L; ++t) wk[i] += dk[t][i] * cx[L - t];
        // phase-2 work of T_X box i at sx: sum_{t=0..m-1} desc_{L-t}(i) * ck[t] + leaves (final)
        for (int64_t i = 0; i < cx[sx]; ++i) {
          for (int t = 0; t < m; ++t) wx[i] += dx[L - t][i] * ck[t];
          wx[i] += dx[L][i];
        }
        auto bk = linear_partition(wk, world);
        auto bx = linear_partition(wx, world);
        int64_t max1 = 0, max2 = 0, maxx = 0;
        // exchange: sender r sends its B(m) rows x (A at L-m not owned by r)
        std::vector<int64_t> a_own(world, 0);
        for (int r = 0; r < world; ++r) {
          int64_t s1 = 0, s2 = 0;
          for (int64_t i = bk[r]; i < bk[r + 1]; ++i) s1 += wk[i];
          for (int64_t i = bx[r]; i < bx[r + 1]; ++i) s2 += wx[i];
          max1 = std::max(max1, s1);
          max2 = std::max(max2, s2);
          for (int64_t i = bx[r]; i < bx[r + 1]; ++i) a_own[r] += dx[L - m][i];
        }
        for (int r = 0; r < world; ++r) {
          int64_t nb = 0;
          for (int64_t i = bk[r]; i < bk[r + 1]; ++i) nb += dk[m][i];
          int64_t sent = nb * (cx[L - m] - a_own[r]);
          int64_t recv = a_own[r] * (ck[m] - nb);
          maxx = std::max(maxx, std::max(sent, recv));
        }
        int64_t total = max1 + max2 + 4 * maxx;
        if (best_total < 0 || total < best_total) {
          best_total = total;
          best.sk = sk;
          best.sx = sx;
          best.m = m;
          best.k_lo.assign(bk.begin(), bk.end() - 1);
          best.k_hi.assign(bk.begin() + 1, bk.end());
          best.x_lo.assign(bx.begin(), bx.end() - 1);
          best.x_hi.assign(bx.begin() + 1, bx.end());
          if (best_cost) {
            best_cost[0] = max1;
            best_cost[1] = max2;
            best_cost[2] = maxx;
          }
        }
      }
    }
  }
  return best_total < 0 ? SFT_E_ARG : SFT_OK;
}

extern "C" int sft_choose_partition(int L, int world, const int64_t* counts_x, const int64_t* counts_k,
                                    const int32_t* const* parent_x, const int32_t* const* parent_k, int force_sk,
                                    int force_sx, int force_m, int64_t* out, int64_t* out_cost) {
  if (L < 1 || L > 20 || world < 1 || !counts_x || !counts_k || !parent_x || !parent_k || !out)
    return fail(SFT_E_ARG, "sft_choose_partition: bad arguments");
  std::vector<int64_t> cx(counts_x, counts_x + L + 1), ck(counts_k, counts_k + L + 1);
  std::vector<std::vector<int32_t>> px(L + 1), pk(L + 1);
  for (int l = 1; l <= L; ++l) {
    px[l].assign(parent_x[l], parent_x[l] + cx[l]);
    pk[l].assign(parent_k[l], parent_k[l] + ck[l]);
  }
  Partition part;
  int rc = choose_partition(L, world, cx, ck, px, pk, force_sk, force_sx, force_m, part, out_cost);
  if (rc) return fail(rc, "sft_choose_partition: no feasible (s_K, s_X, m)");
  out[0] = part.sk;
  out[1] = part.sx;
  out[2] = part.m;
  for (int r = 0; r < world; ++r) {
    out[3 + 4 * r] = part.k_lo[r];
    out[4 + 4 * r] = part.k_hi[r];
    out[5 + 4 * r] = part.x_lo[r];
    out[6 + 4 * r] = part.x_hi[r];
  }
  return SFT_OK;
}

static LevelDims level_dims(const sft_plan_s* P, int t) {
  const int L = P->L;
  LevelDims ld;
  ld.t = t;
  ld.cbK = P->K.lev[t].child_begin;
  ld.mK = P->K.lev[t].child_mask;
  ld.cbX = P->X.lev[L - t - 1].child_begin;
  ld.mX = P->X.lev[L - t - 1].child_mask;
  ld.seg = nullptr;
  ld.nseg = 0;
  return ld;
}

// Phase-1 style level (B restricted to this rank's T_K range, all A).
static LevelDims level_dims_k(const sft_plan_s* P, int t) {
  const int L = P->L;
  LevelDims ld = level_dims(P, t);
  ld.b_lo = P->k_rng[t].lo;
  ld.b_hi = P->k_rng[t].hi;
  ld.ap_lo = 0;
  ld.ap_hi = P->X.counts[L - t - 1];
  ld.in_b0 = P->k_rng[t + 1].lo;
  ld.in_nA = P->X.counts[L - t - 1];
  ld.in_a0 = 0;
  ld.out_b0 = P->k_rng[t].lo;
  ld.out_nA = P->X.counts[L - t];
  ld.out_a0 = 0;
  return ld;
}

// Phase-2 style level (all B, A restricted to this rank's T_X range).
static LevelDims level_dims_x(const sft_plan_s* P, int t) {
  const int L = P->L;
  LevelDims ld = level_dims(P, t);
  ld.b_lo = 0;
  ld.b_hi = P->K.counts[t];
  ld.ap_lo = P->x_rng[L - t - 1].lo;
  ld.ap_hi = P->x_rng[L - t - 1].hi;
  ld.in_b0 = 0;
  ld.in_nA = P->x_rng[L - t - 1].hi - P->x_rng[L - t - 1].lo;
  ld.in_a0 = P->x_rng[L - t - 1].lo;
  ld.out_b0 = 0;
  ld.out_nA = P->x_rng[L - t].hi - P->x_rng[L - t].lo;
  ld.out_a0 = P->x_rng[L - t].lo;
  return ld;
}

// The dims of level t exactly as the apply calls use them (sft_apply, or the
// two phases of a multi-rank plan, with the exchange layout at level m).
static LevelDims apply_dims(const sft_plan_s* P, int t) {
  if (!P->sharded) return level_dims_k(P, t);
  if (t >= P->part.m) {
    LevelDims ld = level_dims_k(P, t);
    if (t == P->part.m) {
      ld.seg = P->d_seg;
      ld.nseg = P->world;
    }
    return ld;
  }
  return level_dims_x(P, t);
}

// Two-level launch with output level t (world 1, 2D): super-groups (A'', B),
// B at level t, A'' at level L-t-2; input = level t+2 pairs, output = level t.
static LevelDims two_level_dims(const sft_plan_s* P, int t) {
  const int L = P->L;
  LevelDims ld = level_dims_k(P, t);
  ld.f2 = 1;
  ld.ap_lo = 0;
  ld.ap_hi = P->X.counts[L - t - 2];
  ld.in_b0 = 0;
  ld.in_nA = P->X.counts[L - t - 2];
  ld.in_a0 = 0;
  ld.cbK1 = P->K.lev[t + 1].child_begin;
  ld.mK1 = P->K.lev[t + 1].child_mask;
  ld.cbX2 = P->X.lev[L - t - 2].child_begin;
  ld.mX2 = P->X.lev[L - t - 2].child_mask;
  return ld;
}

// Dims of the translation launch whose output level is t (two-level or single)
static LevelDims launch_dims(const sft_plan_s* P, int t) {
  const bool f2 = t < (int)P->launch_f2_out.size() && P->launch_f2_out[t];
  LevelDims ld = f2 ? two_level_dims(P, t) : apply_dims(P, t);
  ld.ctr = P->tctr ? P->tctr + 2 * t : nullptr;
  return ld;
}

static LevelDims apply_dims_sched(const sft_plan_s* P, int t) {
  LevelDims ld = launch_dims(P, t);
  ld.sched = P->sched ? P->sched + P->sched_off[t] : nullptr;
  return ld;
}

// ---------------------------------------------------------------------------
// plan
// ---------------------------------------------------------------------------
// Event pool: plans are created and destroyed per step in the bench (and in
// serving loops); cudaEventCreate/Destroy cost several microseconds of host
// time each, on the plan's critical path.  Events are recycled instead (a
// re-recorded event is safe: stream waits capture the event's state at the
// time of the wait call).
// (events belong to a device: one pool per device and kind)
static std::mutex g_ev_mu;
static std::map<int, std::vector<cudaEvent_t>> g_ev_pool[2];  // [0] timing, [1] cudaEventDisableTiming
static int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}
static cudaEvent_t ev_get(bool timing) {
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lk(g_ev_mu);
    auto& v = g_ev_pool[timing ? 0 : 1][dev];
    if (!v.empty()) {
      cudaEvent_t e = v.back();
      v.pop_back();
      return e;
    }
  }
  cudaEvent_t e = nullptr;
  cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming);
  return e;
}
static void ev_put(cudaEvent_t e, bool timing, int dev) {
  if (!e) return;
  std::lock_guard<std::mutex> lk(g_ev_mu);
  g_ev_pool[timing ? 0 : 1][dev].push_back(e);
}

// Block cache: the device blocks of destroyed plans (tree arena, level
// buffers, host staging) are kept per device and handed to the next plan of a
// similar size instead of going back to the stream-ordered pool -- measured on
// B200, a cudaMallocAsync of a ~50 MB block costs ~35 us of host time on the
// plan's critical path even when the pool holds the freed block
// (scripts/malloc_async_probe.cu), a reuse from here ~1 us.  A block freed on
// another stream is reused behind an event recorded at its free.
namespace {
struct CachedBlock {
  void* p;
  size_t bytes;
  cudaStream_t s;
  cudaEvent_t ev;
  int dev;
};
std::mutex g_blk_mu;
std::vector<CachedBlock> g_blk;
constexpr int kBlkPerDev = 8;
}  // namespace

namespace sft {
cudaError_t block_alloc(void** out, size_t bytes, cudaStream_t s) {
  const int dev = current_device();
  {
    std::lock_guard<std::mutex> lk(g_blk_mu);
    int best = -1;
    for (int i = 0; i < (int)g_blk.size(); ++i) {
      const CachedBlock& b = g_blk[i];
      if (b.dev != dev || b.bytes < bytes || b.bytes > bytes + bytes / 4 + (1u << 20)) continue;
      if (best < 0 || b.bytes < g_blk[best].bytes) best = i;
    }
    if (best >= 0) {
      CachedBlock b = g_blk[best];
      g_blk.erase(g_blk.begin() + best);
      cudaError_t e = b.s == s ? cudaSuccess : cudaStreamWaitEvent(s, b.ev, 0);
      ev_put(b.ev, false, dev);
      if (e != cudaSuccess) return e;
      *out = b.p;
      return cudaSuccess;
    }
  }
  return cudaMallocAsync(out, bytes, s);
}

void block_free(void* p, size_t bytes, cudaStream_t s) {
  if (!p) return;
  const int dev = current_device();
  cudaEvent_t ev = ev_get(false);
  if (!ev || cudaEventRecord(ev, s) != cudaSuccess) {
    if (ev) ev_put(ev, false, dev);
    cudaFreeAsync(p, s);
    return;
  }
  std::lock_guard<std::mutex> lk(g_blk_mu);
  int ndev = 0, oldest = -1;
  for (int i = 0; i < (int)g_blk.size(); ++i)
    if (g_blk[i].dev == dev) {
      ++ndev;
      if (oldest < 0) oldest = i;
    }
  if (ndev >= kBlkPerDev) {  // evict the oldest of this device (stream-ordered after its own uses)
    CachedBlock b = g_blk[oldest];
    g_blk.erase(g_blk.begin() + oldest);
    cudaStreamWaitEvent(s, b.ev, 0);
    cudaFreeAsync(b.p, s);
    ev_put(b.ev, false, dev);
  }
  g_blk.push_back(CachedBlock{p, bytes, s, ev, dev});
}
}  // namespace sft

static void plan_free(sft_plan_s* P) {
  if (!P) return;
  cudaStream_t s = P->stream;
  if (P->sched_ready) cudaStreamWaitEvent(s, P->sched_ready, 0);
  free_tree(P->X, s);
  free_tree(P->K, s);
  if (P->buf[0]) block_free(P->buf[0], P->blk_bytes, s);  // one block: both level buffers (+ schedules)
  for (int i = 0; i < 2; ++i)
    if (P->bufb[i]) cudaFreeAsync(P->bufb[i], s);
  if (P->f_stage) block_free(P->f_stage, P->f_stage_bytes, s);
  if (P->u_stage) block_free(P->u_stage, P->u_stage_bytes, s);
  if (P->d_seg) cudaFreeAsync(P->d_seg, s);
  for (void* q : {(void*)P->xsend, (void*)P->xrecv, (void*)P->u_all, (void*)P->d_ubounds})
    if (q) cudaFreeAsync(q, s);
  for (int i = 0; i < P->ev_created; ++i) cudaEventDestroy(P->ev[i]);
  if (P->f_copied) cudaEventDestroy(P->f_copied);
  for (int i = 0; i < 2; ++i) ev_put(P->plan_ev[i], true, P->dev);
  ev_put(P->sched_fork, false, P->dev);
  ev_put(P->sched_ready, false, P->dev);
  ev_put(P->sched_first, false, P->dev);
  // no sync: the frees above are stream-ordered behind any pending work
  delete P;
}

// SFT_PLAN_TRACE=1: host timestamps (us since entry) of sft_plan's milestones on
// stderr; marks with dev = true also write the GPU's %globaltimer from a
// one-thread kernel on the plan stream (device times relative to the first)
__global__ void k_stamp(unsigned long long* out) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  *out = t;
}
struct PlanTrace {
  bool on = false;
  std::chrono::steady_clock::time_point t0;
  char buf[1024];
  int n = 0;
  unsigned long long* d_ts = nullptr;
  const char* evn[16];
  int nev = 0;
  PlanTrace() {
    const char* e = getenv("SFT_PLAN_TRACE");
    on = e && e[0] == '1';
    t0 = std::chrono::steady_clock::now();
    // device memory (a managed page would fault on each first GPU write and
    // skew the stamps by ~30 us)
    if (on) cudaMalloc(&d_ts, 16 * sizeof(unsigned long long));
  }
  void mark(const char* what, cudaStream_t s, bool dev) {
    if (!on || n > 900) return;
    const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
    n += snprintf(buf + n, sizeof(buf) - n, " %s=%.1f", what, us);
    if (dev && nev < 16 && d_ts) {
      k_stamp<<<1, 1, 0, s>>>(d_ts + nev);
      evn[nev++] = what;
    }
  }
  ~PlanTrace() {
    if (!on) return;
    fprintf(stderr, "[sft_plan] host us:%s\n", buf);
    if (nev) {
      unsigned long long h[16];
      cudaDeviceSynchronize();
      cudaMemcpy(h, d_ts, nev * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      fprintf(stderr, "[sft_plan] device us:");
      for (int i = 0; i < nev; ++i) fprintf(stderr, " %s=%.1f", evn[i], (h[i] - h[0]) * 1e-3);
      fprintf(stderr, "\n");
    }
    cudaFree(d_ts);
    cudaGetLastError();
  }
};
static thread_local PlanTrace* g_trace = nullptr;
namespace sft {
void trace_mark(const char* what, cudaStream_t s, bool dev) {
  if (g_trace) g_trace->mark(what, s, dev);
}
}  // namespace sft

// two-level launches by default for plans whose largest level has fewer pairs (see sft_plan)
constexpr int64_t kF2MaxPairs = 32768;

static int supported_p(int d, int p) { return (d == 2 || d == 3) && (p == 5 || p == 7 || p == 9); }

extern "C" int sft_plan(int dim, int64_t N, int p, const double* x, int64_t nx, const double* k, int64_t nk,
                        const sft_opts* opts, sft_plan_t* out) {
  PlanTrace trace;
  g_trace = trace.on ? &trace : nullptr;
  struct Untrace {
    ~Untrace() { g_trace = nullptr; }
  } untrace;
  if (!out) return fail(SFT_E_ARG, "out is NULL");
  if (dim != 2 && dim != 3) return fail(SFT_E_ARG, "dim must be 2 or 3");
  if (N < 2 || N > (1 << 20) || (N & (N - 1))) return fail(SFT_E_ARG, "N must be a power of two in [2, 2^20]");
  if (!supported_p(dim, p)) return fail(SFT_E_ARG, "p must be 5, 7 or 9");
  if (nx < 1 || nk < 1 || nx > INT32_MAX || nk > INT32_MAX) return fail(SFT_E_ARG, "point counts must be >= 1");
  if (!x || !k) return fail(SFT_E_ARG, "x or k is NULL");
  sft_opts o;
  sft_default_opts(&o);
  if (opts) o = *opts;
  if (o.precision != 0 && o.precision != 1) return fail(SFT_E_ARG, "precision must be 0 (FP64) or 1 (FP32)");
  if (o.world < 1 || o.rank < 0 || o.rank >= o.world) return fail(SFT_E_ARG, "bad rank/world");
  const bool sharded = o.world > 1 || (o.nccl_id != nullptr && o.exchange_level >= 0);
  if (o.precision == 1 && sharded) return fail(SFT_E_ARG, "the FP32 variant is single-GPU (world == 1)");
  if (o.adjoint && sharded) return fail(SFT_E_ARG, "the adjoint plan is single-GPU (world == 1)");
  if (o.adjoint) {
    // adjoint = conj o forward(targets k, sources x) o conj: swap the point sets
    std::swap(x, k);
    std::swap(nx, nk);
  }
  sft_plan_s* P = new (std::nothrow) sft_plan_s();
  if (!P) return fail(SFT_E_NOMEM, "host allocation failed");
  P->conj = o.adjoint ? 1 : 0;
  P->d = dim;
  P->p = p;
  P->N = N;
  int L = 0;
  while ((int64_t(1) << L) < N) ++L;
  P->L = L;
  P->nx = nx;
  P->nk = nk;
  P->rank = o.rank;
  P->world = o.world;
  // sharded path: world > 1, or one rank forced onto it (nccl_id and an
  // explicit exchange level: the exchange machinery on a single GPU)
  P->sharded = sharded;
  P->prec = o.precision;
  {
    const int64_t pd = ipow64(p, dim);
    P->pds = pair_stride((int)pd, P->prec);  // FP32 (and SFT_PAD_EVEN): 16 / 32-byte multiple per array
  }
  P->stream = (cudaStream_t)o.stream;
  P->dev = current_device();
  cudaStream_t s = P->stream;

  // stream-ordered allocations: keep freed memory in the pool so plan/destroy
  // cycles do not go back to the driver
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  std::string err;
  P->tab = get_device_tables(p, &err);
  if (!P->tab) {
    delete P;
    return fail(SFT_E_CUDA, err);
  }
  cudaEvent_t e0 = ev_get(true), e1 = ev_get(true);
  cudaEventRecord(e0, s);
  // taken now (host time overlaps the tree build), used after the counts sync
  P->sched_fork = ev_get(false);
  P->sched_ready = ev_get(false);
  P->sched_first = ev_get(false);
  bool sched_recorded = false;
  auto bail = [&](int code, const std::string& m) {
    if (!P->plan_ev[0]) {
      ev_put(e0, true, P->dev);
      ev_put(e1, true, P->dev);
    }
    if (!sched_recorded) {  // plan_free waits on sched_ready: never on an unrecorded pooled event
      ev_put(P->sched_fork, false, P->dev);
      ev_put(P->sched_ready, false, P->dev);
      ev_put(P->sched_first, false, P->dev);
      P->sched_fork = P->sched_ready = P->sched_first = nullptr;
    }
    plan_free(P);
    return fail(code, m);
  };

  // stage host coordinates
  const double* xd = x;
  const double* kd = k;
  double* xs = nullptr;
  double* ks = nullptr;
  if (!is_device_ptr(x)) {
    if (cudaMallocAsync(&xs, nx * dim * sizeof(double), s) != cudaSuccess) return bail(SFT_E_NOMEM, "alloc x");
    cudaMemcpyAsync(xs, x, nx * dim * sizeof(double), cudaMemcpyHostToDevice, s);
    xd = xs;
  }
  if (!is_device_ptr(k)) {
    if (cudaMallocAsync(&ks, nk * dim * sizeof(double), s) != cudaSuccess) return bail(SFT_E_NOMEM, "alloc k");
    cudaMemcpyAsync(ks, k, nk * dim * sizeof(double), cudaMemcpyHostToDevice, s);
    kd = ks;
  }
  trace_mark("pre_tree", s, true);
  int rc = build_trees(P, xd, kd, &err);
  trace_mark("trees", s, true);
  if (xs) cudaFreeAsync(xs, s);
  if (ks) cudaFreeAsync(ks, s);
  if (rc) return bail(rc, err);

  // level buffers: max over t of (local) pairs(t)
  const int64_t PD = ipow64(p, dim);
  if (P->sharded) {
    // partition + per-rank ranges; needs parent arrays on the host
    std::vector<std::vector<int32_t>> px(L + 1), pk(L + 1);
    for (int l = 1; l <= L; ++l) {
      px[l].resize(P->X.counts[l]);
      pk[l].resize(P->K.counts[l]);
      cudaMemcpyAsync(px[l].data(), P->X.lev[l].parent, px[l].size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      cudaMemcpyAsync(pk[l].data(), P->K.lev[l].parent, pk[l].size() * sizeof(int32_t), cudaMemcpyDeviceToHost, s);
    }
    if (cudaStreamSynchronize(s) != cudaSuccess) return bail(SFT_E_CUDA, "sync");
    int64_t cost[3];
    if (choose_partition(L, P->world, P->X.counts, P->K.counts, px, pk, o.split_k, o.split_x, o.exchange_level,
                         P->part, cost))
      return bail(SFT_E_ARG, "no feasible partition for the requested split levels");
    const Partition& pt = P->part;
    descend_ranges(pk, pt.sk, pt.k_lo[P->rank], pt.k_hi[P->rank], L, P->k_rng);
    descend_ranges(px, pt.sx, pt.x_lo[P->rank], pt.x_hi[P->rank], L, P->x_rng);
    {
      int32_t fp[2] = {0, 0};
      cudaMemcpy(&fp[0], P->X.first_pt + P->x_rng[L].lo, sizeof(int32_t), cudaMemcpyDeviceToHost);
      cudaMemcpy(&fp[1], P->X.first_pt + P->x_rng[L].hi, sizeof(int32_t), cudaMemcpyDeviceToHost);
      P->x_pt_lo = fp[0];
      P->x_pt_hi = fp[1];
      cudaMemcpy(&fp[0], P->K.first_pt + P->k_rng[L].lo, sizeof(int32_t), cudaMemcpyDeviceToHost);
      cudaMemcpy(&fp[1], P->K.first_pt + P->k_rng[L].hi, sizeof(int32_t), cudaMemcpyDeviceToHost);
      P->k_src_lo = fp[0];
      P->k_src_hi = fp[1];
    }
    // exchange layout at level m: A boundaries at level L-m for every rank
    const int m = pt.m, W = P->world;
    std::vector<int64_t> abound(W + 1), nb_of(W);
    std::vector<LevelRange> tmp;
    for (int q = 0; q < W; ++q) {
      descend_ranges(px, pt.sx, pt.x_lo[q], pt.x_hi[q], L, tmp);
      abound[q] = tmp[L - m].lo;
      abound[q + 1] = tmp[L - m].hi;
      descend_ranges(pk, pt.sk, pt.k_lo[q], pt.k_hi[q], L, tmp);
      nb_of[q] = tmp[m].hi - tmp[m].lo;
    }
    const int64_t my_nb = P->k_rng[m].hi - P->k_rng[m].lo;
    const int64_t my_na = abound[P->rank + 1] - abound[P->rank];
    P->send_counts.assign(W, 0);
    P->recv_counts.assign(W, 0);
    std::vector<int64_t> seg(2 * W + 1, 0);
    int64_t base = 0;
    for (int q = 0; q < W; ++q) {
      seg[q] = abound[q];
      seg[W + 1 + q] = base;  // pair offset of segment q in the send buffer
      P->send_counts[q] = my_nb * (abound[q + 1] - abound[q]) * PD;
      P->recv_counts[q] = nb_of[q] * my_na * PD;
      base += my_nb * (abound[q + 1] - abound[q]);
    }
    seg[W] = abound[W];
    // fused exchange: offset (elements) of this rank's segment in every
    // receiver's buffer (receivers concatenate the senders' segments in rank order)
    P->seg_host = seg;
    P->peer_off.assign(W, 0);
    for (int q = 0; q < W; ++q) {
      const int64_t na_q = abound[q + 1] - abound[q];
      int64_t o = 0;
      for (int r = 0; r < P->rank; ++r) o += nb_of[r] * na_q;
      P->peer_off[q] = o * PD;
    }
    if (cudaMallocAsync(&P->d_seg, seg.size() * sizeof(int64_t), s) != cudaSuccess) return bail(SFT_E_NOMEM, "seg");
    cudaMemcpyAsync(P->d_seg, seg.data(), seg.size() * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    if (o.nccl_id) {
      // in-library collectives: the communicator (cached per id),
      // the exchange buffers, and the all-gather layout of u -- rank q's targets
      // are the sorted points [xb[q], xb[q+1]) of its T_X subtrees
      std::string nerr;
      if (int nrc = nccl_comm_get(o.nccl_id, o.rank, W, &P->comm, &nerr)) return bail(nrc, nerr);
      int64_t ns = 0, nr = 0;
      for (int q = 0; q < W; ++q) {
        ns += P->send_counts[q];
        nr += P->recv_counts[q];
      }
      std::vector<int64_t> xb(W + 1, 0);
      std::vector<int32_t> fp(W + 1, 0);
      for (int q = 0; q <= W; ++q) {
        descend_ranges(px, pt.sx, q < W ? pt.x_lo[q] : pt.x_hi[W - 1], q < W ? pt.x_hi[q] : pt.x_hi[W - 1], L, tmp);
        cudaMemcpyAsync(&fp[q], P->X.first_pt + tmp[L].lo, sizeof(int32_t), cudaMemcpyDeviceToHost, s);
      }
      if (cudaStreamSynchronize(s) != cudaSuccess) return bail(SFT_E_CUDA, "sync");
      int64_t mxc = 1;
      for (int q = 0; q <= W; ++q) xb[q] = q < W ? fp[q] : nx;
      xb[0] = 0;
      for (int q = 0; q < W; ++q) mxc = std::max(mxc, xb[q + 1] - xb[q]);
      P->u_cnt = mxc;
      P->u_bounds = xb;
      if (cudaMallocAsync(&P->xsend, std::max<int64_t>(ns, 1) * sizeof(double2), s) != cudaSuccess ||
          cudaMallocAsync(&P->xrecv, std::max<int64_t>(nr, 1) * sizeof(double2), s) != cudaSuccess ||
          cudaMallocAsync(&P->u_all, (size_t)(W + 1) * mxc * sizeof(double2), s) != cudaSuccess ||
          cudaMallocAsync(&P->d_ubounds, (W + 1) * sizeof(int64_t), s) != cudaSuccess)
        return bail(SFT_E_NOMEM, "exchange buffers");
      cudaMemcpyAsync(P->d_ubounds, xb.data(), (W + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
      if (cudaStreamSynchronize(s) != cudaSuccess) return bail(SFT_E_CUDA, "sync");  // (xb is a host temporary)
    }
    int64_t mx = 0;
    for (int t = m; t <= L; ++t) mx = std::max(mx, (P->k_rng[t].hi - P->k_rng[t].lo) * P->X.counts[L - t]);
    for (int t = 0; t <= m; ++t) mx = std::max(mx, P->K.counts[t] * (P->x_rng[L - t].hi - P->x_rng[L - t].lo));
    P->buf_elems = (size_t)mx * P->pds;
  } else {
    int64_t mx = 0;
    for (int t = 0; t <= L; ++t) mx = std::max(mx, P->K.counts[t] * P->X.counts[L - t]);
    P->buf_elems = (size_t)mx * P->pds;
    P->k_rng.assign(L + 1, LevelRange());
    P->x_rng.assign(L + 1, LevelRange());
    P->x_pt_lo = 0;
    P->x_pt_hi = nx;
    P->k_src_lo = 0;
    P->k_src_hi = nk;
    for (int l = 0; l <= L; ++l) {
      P->k_rng[l].hi = P->K.counts[l];
      P->x_rng[l].hi = P->X.counts[l];
    }
  }
  // the tile schedules address a level buffer with 32-bit element offsets
  // (TaskRec, group records): reject plans whose largest level does not fit
  // (e.g. 3D N = 1024 p = 9 on dense surfaces) instead of wrapping silently
  if (P->buf_elems >= (size_t(1) << 32))
    return bail(SFT_E_ARG, "a level of this plan holds " + std::to_string(P->buf_elems) +
                               " complex elements; the translation schedules address at most 2^32 - 1");
  // translation launches of the single-GPU apply: two-level launches (levels
  // t+1 and t from t+2) where supported, from the leaf level down; a single
  // level 0 is left when L is odd.  Multi-rank plans run single levels.
  P->launch_t.clear();
  P->launch_f2_out.assign(L, 0);
  {
    // Two-level launches halve the per-level latency chain (load, compute,
    // store, kernel boundary), which is what a small plan's levels cost:
    // measured (B200, round 2) C0 apply 0.039 -> 0.029 ms, C1 0.075 -> 0.066 ms
    // with every pair fused.  On large plans a super-group's stage is half
    // empty (~2 of 4 first-level groups present on curves) and the HBM round
    // trip they save is not the limiter: C2 0.927 -> 1.311 ms (all), 0.939
    // (leaf-end pair only).  Default: every pair fused when the largest level
    // has fewer than kF2MaxPairs pairs, else none; SFT_F2=0|first|all overrides.
    const char* fe = getenv("SFT_F2");
    int64_t max_pairs = 0;
    for (int tt = 0; tt <= L; ++tt) max_pairs = std::max<int64_t>(max_pairs, P->K.counts[tt] * P->X.counts[L - tt]);
    const bool f2_all = fe ? std::string(fe) == "all" : max_pairs < kF2MaxPairs;
    const bool f2 = two_level_supported(P) && (f2_all || (fe && std::string(fe) == "first"));
    int t = L - 1;
    while (t >= 0) {
      if (f2 && t >= 1 && (f2_all || t == L - 1)) {
        P->launch_t.push_back(t - 1);
        P->launch_f2_out[t - 1] = 1;
        t -= 2;
      } else {
        P->launch_t.push_back(t);
        t -= 1;
      }
    }
  }
  // one allocation: level buffer 0 | level buffer 1 | tile schedules of every launch
  // (indexed by the launch's output level; levels consumed inside a two-level launch have none)
  {
    P->sched_off.assign(L + 1, 0);
    size_t tot = 0;
    for (int t = 0; t < L; ++t) {
      P->sched_off[t] = tot;
      const bool inner = t >= 1 && P->launch_f2_out[t - 1];  // level t produced inside a two-level launch
      if (!inner) tot += (schedule_bytes(P, launch_dims(P, t)) + 255) / 256 * 256;
    }
    P->sched_off[L] = tot;
    // dynamic tile scheduling (SFT_DYN=0: static grid-stride assignment)
    const char* dyn = getenv("SFT_DYN");
    const size_t cb = (tot > 0 && !(dyn && dyn[0] == '0')) ? ((size_t)2 * L * sizeof(int) + 255) / 256 * 256 : 0;
    const size_t bb = (P->buf_elems * (P->prec == 1 ? sizeof(float2) : sizeof(double2)) + 255) / 256 * 256;
    char* blk = nullptr;
    if (block_alloc((void**)&blk, 2 * bb + tot + cb, s) != cudaSuccess)
      return bail(SFT_E_NOMEM, "level buffer allocation failed");
    P->blk_bytes = 2 * bb + tot + cb;
    P->buf[0] = (double2*)blk;
    P->buf[1] = (double2*)(blk + bb);
    P->sched = tot > 0 ? (unsigned char*)(blk + 2 * bb) : nullptr;
    P->tctr = cb > 0 ? (int*)(blk + 2 * bb + tot) : nullptr;
    trace_mark("bufs");
    if (tot > 0) {
      // the first translation launch's schedule first (its own event: the
      // first translation waits only for it), then all the others
      std::vector<LevelDims> dims;
      std::vector<unsigned char*> dst;
      // (only when the first launch is a two-level one: its schedule kernel is
      // a separate launch anyway)
      // (a separate first-launch schedule only pays when the schedules are long)
      const int t_first = !P->sharded && !P->launch_t.empty() && P->launch_f2_out[P->launch_t[0]] &&
                                  P->K.counts[L] * P->X.counts[0] >= kF2MaxPairs
                              ? P->launch_t[0]
                              : -1;
      for (int t = 0; t < L; ++t) {
        if (t >= 1 && P->launch_f2_out[t - 1]) continue;
        if (t == t_first) continue;
        dims.push_back(launch_dims(P, t));
        dst.push_back(P->sched + P->sched_off[t]);
      }
      // the schedules are built on a side stream so that they overlap the
      // first kernels of the apply (the leaf kernel needs only the trees);
      // the first translation waits on sched_ready
      cudaStream_t side = side_stream();
      cudaEventRecord(P->sched_fork, s);
      cudaStreamWaitEvent(side, P->sched_fork, 0);
      cudaError_t ce = cudaSuccess;
      if (t_first >= 0) {
        const LevelDims d0 = launch_dims(P, t_first);
        unsigned char* d0dst = P->sched + P->sched_off[t_first];
        ce = launch_schedule(P, &d0, 1, &d0dst, side);
        cudaEventRecord(P->sched_first, side);
      }
      if (ce == cudaSuccess) ce = launch_schedule(P, dims.data(), (int)dims.size(), dst.data(), side);
      cudaEventRecord(P->sched_ready, side);
      sched_recorded = true;
      if (ce != cudaSuccess) return bail(SFT_E_CUDA, std::string("schedule: ") + cudaGetErrorString(ce));
      const char* chk = getenv("SFT_CHECK_SCHED");
      if (chk && chk[0] == '1') {
        cudaStreamWaitEvent(s, P->sched_ready, 0);
        // debug: every level's schedule against its buffer sizes
        for (int t = 0; t < L; ++t) {
          if (t >= 1 && P->launch_f2_out[t - 1]) continue;
          const LevelDims ld = launch_dims(P, t);
          const int64_t in_pairs = (int64_t)(P->buf_elems / P->pds), out_pairs = in_pairs;
          cudaError_t ce = check_schedule(P, ld, P->sched + P->sched_off[t], in_pairs, out_pairs, P->d_err);
          if (ce != cudaSuccess) return bail(SFT_E_CUDA, std::string("check: ") + cudaGetErrorString(ce));
        }
        int herr = 0;
        cudaStreamWaitEvent(s, P->sched_ready, 0);
        cudaMemcpyAsync(&herr, P->d_err, sizeof(int), cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
        if (herr & 4) return bail(SFT_E_CUDA, "tile schedule failed its invariants");
      }
    }
  }
  if (!sched_recorded) {  // no schedule kernel (no translation groups / non-ws kernel)
    ev_put(P->sched_fork, false, P->dev);
    ev_put(P->sched_ready, false, P->dev);
    ev_put(P->sched_first, false, P->dev);
    P->sched_fork = P->sched_ready = P->sched_first = nullptr;
    sched_recorded = true;
  }
  if (P->sharded || P->launch_t.empty() || !P->launch_f2_out[P->launch_t[0]]) {  // launch 0 waits on sched_ready
    ev_put(P->sched_first, false, P->dev);
    P->sched_first = nullptr;
  }
  trace_mark("sched");
  // no sync here: the schedule kernel runs behind the caller's next launches;
  // the plan's device time is read lazily (sft_plan_stats)
  cudaEventRecord(e1, s);
  P->plan_ev[0] = e0;
  P->plan_ev[1] = e1;
  P->plan_ms = -1.0;
  cudaError_t ce = cudaGetLastError();
  if (ce != cudaSuccess) {
    plan_free(P);
    return fail(SFT_E_CUDA, cudaGetErrorString(ce));
  }
  *out = P;
  return SFT_OK;
}

// Far-field adapter (eq. far): u_inf(xhat_i) = sum_j e^{-i kappa xhat_i . y_j} F_j.
// With N = the smallest power of two >= max(2, kappa/pi), x = N/2 - kappa xhat/(2 pi) and
// k = N y lie in [0,N]^d and 2 pi x.k/N = pi sum_a k_a - kappa xhat.y ("after we rescale
// xhat and y by a factor of N, (far) takes the form of (sfft)").  The leftover
// phase e^{i pi sum_a k_a} is folded into the leaf kernel (forward: a sign per leaf) or the
// final kernel (adjoint); the butterfly itself is unchanged.
extern "C" int sft_farfield_plan(int dim, double kappa, int p, const double* xhat, int64_t nx, const double* y,
                                 int64_t ny, const sft_opts* opts, sft_plan_t* out) {
  if (!out) return fail(SFT_E_ARG, "out is NULL");
  if (dim != 2 && dim != 3) return fail(SFT_E_ARG, "dim must be 2 or 3");
  if (!(kappa > 0.0) || !std::isfinite(kappa) || kappa > 3.14159265358979323846 * (1 << 20))
    return fail(SFT_E_ARG, "kappa must be in (0, pi * 2^20]");
  if (!xhat || !y) return fail(SFT_E_ARG, "xhat or y is NULL");
  if (nx < 1 || ny < 1 || nx > INT32_MAX || ny > INT32_MAX) return fail(SFT_E_ARG, "point counts must be >= 1");
  if (opts && opts->world != 1) return fail(SFT_E_ARG, "the far-field plan is single-GPU (world == 1)");
  int64_t N = 2;
  while ((double)N < kappa / 3.14159265358979323846) N <<= 1;
  cudaStream_t s = opts ? (cudaStream_t)opts->stream : nullptr;
  double *dx = nullptr, *dk = nullptr, *dxh = nullptr, *dy = nullptr;
  auto cleanup = [&]() {
    for (double* q : {dx, dk, dxh, dy})
      if (q) cudaFreeAsync(q, s);
  };
  const size_t bx = (size_t)nx * dim * sizeof(double), by = (size_t)ny * dim * sizeof(double);
  if (cudaMallocAsync(&dx, bx, s) != cudaSuccess || cudaMallocAsync(&dk, by, s) != cudaSuccess) {
    cudaGetLastError();
    cleanup();
    return fail(SFT_E_NOMEM, "far-field coordinate buffers");
  }
  const double* sx = xhat;
  const double* sy = y;
  if (!is_device_ptr(xhat)) {
    if (cudaMallocAsync(&dxh, bx, s) != cudaSuccess) { cleanup(); return fail(SFT_E_NOMEM, "xhat staging"); }
    cudaMemcpyAsync(dxh, xhat, bx, cudaMemcpyHostToDevice, s);
    sx = dxh;
  }
  if (!is_device_ptr(y)) {
    if (cudaMallocAsync(&dy, by, s) != cudaSuccess) { cleanup(); return fail(SFT_E_NOMEM, "y staging"); }
    cudaMemcpyAsync(dy, y, by, cudaMemcpyHostToDevice, s);
    sy = dy;
  }
  cudaError_t ce = launch_ff_coords(sx, nx, sy, ny, dim, kappa, N, dx, dk, s);
  if (ce != cudaSuccess) {
    cleanup();
    return fail(SFT_E_CUDA, cudaGetErrorString(ce));
  }
  sft_plan_t P = nullptr;
  const int rc = sft_plan(dim, N, p, dx, nx, dk, ny, opts, &P);
  cleanup();  // stream-ordered: sft_plan has consumed (copied) the coordinates
  if (rc != SFT_OK) return rc;
  P->ffmod = 1;
  *out = P;
  return SFT_OK;
}

extern "C" int sft_destroy(sft_plan_t plan) {
  plan_free(plan);
  return SFT_OK;
}

// ---------------------------------------------------------------------------
// apply
// ---------------------------------------------------------------------------
static void tmark(sft_plan_s* P) {
  if (!P->timing) return;
  if (P->n_ev < 64) cudaEventRecord(P->ev[P->n_ev++], P->stream);
}

// Host f: the staging copy is stream-ordered; sft.h promises that the caller
// may modify or free f once sft_apply returns, so the call waits for the copy
// (not for the kernels queued behind it) before returning.
static cudaError_t f_copy_mark(sft_plan_s* P) {
  if (!P->f_copied) {
    cudaError_t e = cudaEventCreateWithFlags(&P->f_copied, cudaEventDisableTiming);
    if (e != cudaSuccess) return e;
  }
  return cudaEventRecord(P->f_copied, P->stream);
}
static cudaError_t f_copy_wait(sft_plan_s* P) { return cudaEventSynchronize(P->f_copied); }

// tl: output level of each timed translation launch (nullptr: n_levels_first - i);
// a two-level launch's time is booked on its output level (the inner level shows 0)
static int finish_timing(sft_plan_s* P, int n_levels_first, const std::vector<int>* tl = nullptr) {
  if (!P->timing) return SFT_OK;
  CKR(cudaEventSynchronize(P->ev[P->n_ev - 1]));
  // events: [0] start, [1] after leaf, [2..] after each level, [n-1] after final
  float ms;
  P->level_ms.assign(P->L, 0.0);
  double trans = 0;
  cudaEventElapsedTime(&ms, P->ev[0], P->ev[1]);
  P->last_ms[0] = ms;
  int nlev = P->n_ev - 3;
  for (int i = 0; i < nlev; ++i) {
    cudaEventElapsedTime(&ms, P->ev[1 + i], P->ev[2 + i]);
    const int t = tl ? (i < (int)tl->size() ? (*tl)[i] : -1) : n_levels_first - i;
    if (P->timing == 1 && t >= 0 && t < P->L) P->level_ms[t] = ms;  // (mode 2: one chain interval)
    trans += ms;
  }
  P->last_ms[1] = trans;
  cudaEventElapsedTime(&ms, P->ev[P->n_ev - 2], P->ev[P->n_ev - 1]);
  P->last_ms[2] = ms;
  cudaEventElapsedTime(&ms, P->ev[0], P->ev[P->n_ev - 1]);
  P->last_ms[3] = ms;
  return SFT_OK;
}

// Steps 2-4 for nrhs charge vectors (f + r*ldf -> u + r*ldu, complex128
// elements).  nrhs == 1 uses the plan's two level buffers; a batch uses
// [nrhs][buf_elems] buffers (grown on demand) and one launch per step for all
// vectors: the leaf weights, final-step powers, tile schedules and operator
// fragments are computed / read once for every RHS.
static int apply_impl(sft_plan_s* P, int nrhs, const void* f, int64_t ldf, void* u, int64_t ldu) {
  cudaStream_t s = P->stream;
  const int L = P->L;
  const double2* fd = (const double2*)f;
  double2* ud = (double2*)u;
  const bool f_host = !is_device_ptr(f), u_host = !is_device_ptr(u);
  if ((f_host || u_host) && P->stage_rhs < nrhs) {
    if (P->f_stage) block_free(P->f_stage, P->f_stage_bytes, s);
    if (P->u_stage) block_free(P->u_stage, P->u_stage_bytes, s);
    P->f_stage = P->u_stage = nullptr;
    P->stage_rhs = 0;
    P->f_stage_bytes = (size_t)nrhs * P->nk * sizeof(double2);
    P->u_stage_bytes = (size_t)nrhs * P->nx * sizeof(double2);
    CKR(block_alloc((void**)&P->f_stage, P->f_stage_bytes, s));
    CKR(block_alloc((void**)&P->u_stage, P->u_stage_bytes, s));
    P->stage_rhs = nrhs;
  }
  if (f_host) {
    if (ldf == P->nk)  // contiguous: one plain copy (the 2-D path is slower for pinned memory)
      CKR(cudaMemcpyAsync(P->f_stage, f, (size_t)nrhs * P->nk * sizeof(double2), cudaMemcpyHostToDevice, s));
    else
      CKR(cudaMemcpy2DAsync(P->f_stage, P->nk * sizeof(double2), f, ldf * sizeof(double2), P->nk * sizeof(double2),
                            nrhs, cudaMemcpyHostToDevice, s));
    fd = P->f_stage;
    ldf = P->nk;
    CKR(f_copy_mark(P));
  }
  int64_t ldu_dev = ldu;
  if (u_host) {
    ud = P->u_stage;
    ldu_dev = P->nx;
  }
  double2* buf[2] = {P->buf[0], P->buf[1]};
  int64_t rs = 0;
  if (nrhs > 1) {
    if (P->bufb_rhs < nrhs) {
      const size_t esz = P->prec == 1 ? sizeof(float2) : sizeof(double2);
      for (int i = 0; i < 2; ++i) {
        if (P->bufb[i]) cudaFreeAsync(P->bufb[i], s);
        P->bufb[i] = nullptr;
      }
      P->bufb_rhs = 0;
      for (int i = 0; i < 2; ++i)
        if (cudaMallocAsync(&P->bufb[i], (size_t)nrhs * P->buf_elems * esz, s) != cudaSuccess) {
          cudaGetLastError();
          for (int j = 0; j < 2; ++j) {
            if (P->bufb[j]) cudaFreeAsync(P->bufb[j], s);
            P->bufb[j] = nullptr;
          }
          return fail(SFT_E_NOMEM, "batch level buffers: " + std::to_string(nrhs) + " x " +
                                       std::to_string(2.0 * P->buf_elems * esz / 1e9) + " GB");
        }
      P->bufb_rhs = nrhs;
    }
    buf[0] = P->bufb[0];
    buf[1] = P->bufb[1];
    rs = (int64_t)P->buf_elems;
  }
  if (P->timing && P->ev_created < L + 3) {
    for (int i = P->ev_created; i < L + 3; ++i) cudaEventCreate(&P->ev[i]);
    P->ev_created = L + 3;
  }
  P->n_ev = 0;
  tmark(P);
  // step 2: leaf charges, level L buffer
  // the level buffers alternate per launch: leaf -> buf[0], launch i reads
  // buf[i & 1] and writes buf[(i + 1) & 1]
  CKR(launch_leaf(P, fd, buf[0], 0, P->K.counts[L], nrhs, ldf, rs));
  tmark(P);
  // step 3: the translation launches, t = L-1 .. 0 (two-level launches cover
  // levels t+1 and t), after the plan's schedule kernel on the side stream
  const int nl = (int)P->launch_t.size();
  for (int i = 0; i < nl; ++i) {
    // launch 0 needs only its own schedule; the rest were built behind it
    if (i == 0 && P->sched_first) CKR(cudaStreamWaitEvent(s, P->sched_first, 0));
    else if (i <= 1 && P->sched_ready) CKR(cudaStreamWaitEvent(s, P->sched_ready, 0));
    LevelDims ld = apply_dims_sched(P, P->launch_t[i]);
    ld.nrhs = nrhs;
    ld.rs = rs;
    CKR(launch_translate(P, ld, buf[i & 1], buf[(i + 1) & 1]));
    if (P->timing != 2 || i == nl - 1) tmark(P);  // mode 2: the chain as one interval (PDL overlap kept)
  }
  // step 4: final evaluation, level 0 buffer [A leaves]
  CKR(launch_final(P, buf[nl & 1], ud, 0, 0, P->nx, nrhs, rs, ldu_dev));
  tmark(P);
  if (u_host) {
    if (ldu == ldu_dev)
      CKR(cudaMemcpyAsync(u, ud, (size_t)nrhs * P->nx * sizeof(double2), cudaMemcpyDeviceToHost, s));
    else
      CKR(cudaMemcpy2DAsync(u, ldu * sizeof(double2), ud, ldu_dev * sizeof(double2), P->nx * sizeof(double2), nrhs,
                            cudaMemcpyDeviceToHost, s));
    CKR(cudaStreamSynchronize(s));
  } else if (f_host) {
    CKR(f_copy_wait(P));  // the caller may reuse f as soon as we return (sft.h)
  }
  return finish_timing(P, L - 1, &P->launch_t);
}

static int apply_sharded(sft_plan_s* P, const void* f, void* u);

extern "C" int sft_apply(sft_plan_t P, const void* f, void* u) {
  if (!P || !f || !u) return fail(SFT_E_ARG, "NULL argument");
  if (P->sharded) {
    if (!P->comm)
      return fail(SFT_E_STATE, "sharded plan without opts.nccl_id: use the phase calls and your own collective");
    if (!P->peer.empty()) return fail(SFT_E_STATE, "fused-exchange plan: use the phase calls");
    return apply_sharded(P, f, u);
  }
  return apply_impl(P, 1, f, P->nk, u, P->nx);
}

extern "C" int sft_apply_batch(sft_plan_t P, int nrhs, const void* f, int64_t ldf, void* u, int64_t ldu) {
  if (!P || !f || !u) return fail(SFT_E_ARG, "NULL argument");
  if (nrhs < 1 || nrhs > 4096) return fail(SFT_E_ARG, "nrhs must be in [1, 4096]");
  if (ldf < P->nk || ldu < P->nx) return fail(SFT_E_ARG, "ldf >= nk and ldu >= nx required");
  if (P->sharded) return fail(SFT_E_STATE, "sft_apply_batch needs a world == 1 plan");
  return apply_impl(P, nrhs, f, ldf, u, ldu);
}

// ---------------------------------------------------------------------------
// multi-GPU phases
// ---------------------------------------------------------------------------
extern "C" int sft_exchange_counts(sft_plan_t P, int64_t* send_counts, int64_t* recv_counts) {
  if (!P) return fail(SFT_E_ARG, "NULL plan");
  if (!P->sharded) return fail(SFT_E_STATE, "plan is not multi-rank");
  for (int q = 0; q < P->world; ++q) {
    if (send_counts) send_counts[q] = P->send_counts[q];
    if (recv_counts) recv_counts[q] = P->recv_counts[q];
  }
  return SFT_OK;
}

extern "C" int sft_partition_info(sft_plan_t P, int64_t* part) {
  if (!P || !part) return fail(SFT_E_ARG, "NULL argument");
  if (!P->sharded) return fail(SFT_E_STATE, "plan is not multi-rank");
  part[0] = P->part.sk;
  part[1] = P->part.sx;
  part[2] = P->part.m;
  for (int r = 0; r < P->world; ++r) {
    part[3 + 4 * r] = P->part.k_lo[r];
    part[4 + 4 * r] = P->part.k_hi[r];
    part[5 + 4 * r] = P->part.x_lo[r];
    part[6 + 4 * r] = P->part.x_hi[r];
  }
  return SFT_OK;
}

// Timing of the phase calls (sft_set_timing): the translation launches of a
// phase are bracketed by two events; t_ms[1] of sft_last_timing is the sum of
// phase 1 and phase 2 (each phase synchronises its events: diagnostics only)
static void phase_timing_begin(sft_plan_s* P) {
  if (!P->timing) return;
  if (P->ev_created < 2) {
    for (int i = P->ev_created; i < 2; ++i) cudaEventCreate(&P->ev[i]);
    P->ev_created = 2;
  }
  cudaEventRecord(P->ev[0], P->stream);
}
static int phase_timing_end(sft_plan_s* P, bool first) {
  if (!P->timing) return SFT_OK;
  cudaEventRecord(P->ev[1], P->stream);
  CKR(cudaEventSynchronize(P->ev[1]));
  float ms = 0;
  cudaEventElapsedTime(&ms, P->ev[0], P->ev[1]);
  P->last_ms[1] = (first ? 0.0 : P->last_ms[1]) + ms;
  return SFT_OK;
}

// Phase 1 of a sharded plan (levels t = L..m over this rank's T_K subtrees):
// the level-m charges in the send layout at sb, or -- fused exchange -- stored
// straight into the receivers' buffers.  fd: device charges [nk].
static int phase1_run(sft_plan_s* P, const double2* fd, double2* sb) {
  cudaStream_t s = P->stream;
  const int L = P->L, m = P->part.m;
  const bool fused = !P->peer.empty();
  // leaf level: the local leaf range; if m == L the leaf output is the send buffer
  const LevelRange kl = P->k_rng[L];
  if (m == L) {
    // exchange at the leaf level: pairs (A0, B) with the single root A0 of T_X
    // (s_X = 0), so only its owner's segment is non-empty and starts at 0
    double2* out = sb;
    if (fused) {
      int q0 = 0;  // the owner of A0: the only non-empty segment
      for (int q = 0; q < P->world; ++q)
        if (P->seg_host[q + 1] > P->seg_host[q]) q0 = q;
      out = P->peer[q0] + P->peer_off[q0];
    }
    CKR(launch_leaf(P, fd, out, kl.lo, kl.hi));
    if (P->timing) P->last_ms[1] = 0.0;  // no translation in phase 1
    return SFT_OK;
  }
  CKR(launch_leaf(P, fd, P->buf[L & 1], kl.lo, kl.hi));
  if (P->sched_ready) CKR(cudaStreamWaitEvent(s, P->sched_ready, 0));
  phase_timing_begin(P);
  for (int t = L - 1; t >= m; --t) {
    LevelDims ld = apply_dims_sched(P, t);
    double2* out = t == m ? sb : P->buf[t & 1];
    if (t == m && fused) {
      // the exchange level's outputs go straight into the receivers' buffers
      // (NVLink peer stores from the kernel's epilogue): no send buffer, no
      // all-to-all
      ld.npeer = P->world;
      for (int q = 0; q < P->world; ++q) {
        ld.peer[q] = P->peer[q];
        ld.peer_off[q] = P->peer_off[q];
        ld.peer_seg[q] = P->seg_host[P->world + 1 + q];
      }
      ld.peer_seg[P->world] = INT64_MAX;
      out = nullptr;
    }
    CKR(launch_translate(P, ld, P->buf[(t + 1) & 1], out));
  }
  return phase_timing_end(P, true);
}

// Phase 2 (levels t = m-1..0 and step 4 over this rank's T_X subtrees) from
// the received level-m charges.  sorted_out: the potentials of this rank's
// targets in sorted order at ud[0 .. x_pt_hi - x_pt_lo) (the all-gather
// layout); else ud [nx] in user order with every other entry zero.
static int phase2_run(sft_plan_s* P, const double2* in, double2* ud, bool sorted_out) {
  cudaStream_t s = P->stream;
  const int L = P->L, m = P->part.m;
  if (!sorted_out) CKR(launch_zero(ud, P->nx, s));
  if (P->sched_ready) CKR(cudaStreamWaitEvent(s, P->sched_ready, 0));
  phase_timing_begin(P);
  for (int t = m - 1; t >= 0; --t) {
    LevelDims ld = apply_dims_sched(P, t);
    double2* out = P->buf[t & 1];
    CKR(launch_translate(P, ld, in, out));
    in = out;
  }
  if (int rc = phase_timing_end(P, false)) return rc;
  const LevelRange xl = P->x_rng[L];
  CKR(launch_final(P, in, ud, xl.lo, P->x_pt_lo, P->x_pt_hi, 1, 0, 0, sorted_out));
  return SFT_OK;
}

// sft_apply of a sharded plan with an NCCL communicator: phase 1, the level-m
// exchange (grouped ncclSend/ncclRecv), phase 2 into this rank's slot of the
// u all-gather buffer, ncclAllGather, and the scatter to user order -- every
// rank ends with the full u.  All stream-ordered on the
// plan stream.
static int apply_sharded(sft_plan_s* P, const void* f, void* u) {
  cudaStream_t s = P->stream;
  const double2* fd = (const double2*)f;
  const bool f_host = !is_device_ptr(f), u_host = !is_device_ptr(u);
  if (f_host) {
    if (!P->f_stage) {
      P->f_stage_bytes = P->nk * sizeof(double2);
      CKR(block_alloc((void**)&P->f_stage, P->f_stage_bytes, s));
    }
    CKR(cudaMemcpyAsync(P->f_stage, f, P->nk * sizeof(double2), cudaMemcpyHostToDevice, s));
    CKR(f_copy_mark(P));
    fd = P->f_stage;
  }
  double2* ud = (double2*)u;
  if (u_host) {
    if (!P->u_stage) {
      P->u_stage_bytes = P->nx * sizeof(double2);
      CKR(block_alloc((void**)&P->u_stage, P->u_stage_bytes, s));
    }
    ud = P->u_stage;
  }
  std::string err;
  if (int rc = phase1_run(P, fd, P->xsend)) return rc;
  if (int rc = nccl_exchange(P->comm, P->xsend, P->send_counts.data(), P->xrecv, P->recv_counts.data(), P->world, s,
                             &err))
    return fail(rc, err);
  double2* mine = P->u_all + (int64_t)P->rank * P->u_cnt;
  if (int rc = phase2_run(P, P->xrecv, mine, true)) return rc;
  if (int rc = nccl_allgather(P->comm, mine, P->u_all, P->u_cnt, s, &err)) return fail(rc, err);
  CKR(launch_unsort(P->u_all, P->u_cnt, P->d_ubounds, P->world, P->X.perm, ud, P->nx, s));
  if (u_host) {
    CKR(cudaMemcpyAsync(u, ud, P->nx * sizeof(double2), cudaMemcpyDeviceToHost, s));
    CKR(cudaStreamSynchronize(s));
  } else if (f_host) {
    CKR(f_copy_wait(P));
  }
  return SFT_OK;
}

extern "C" int sft_apply_phase1(sft_plan_t P, const void* f, void* sendbuf) {
  if (!P || !f || (!sendbuf && P->peer.empty())) return fail(SFT_E_ARG, "NULL argument");
  if (!P->sharded) return fail(SFT_E_STATE, "plan is not multi-rank");
  if (sendbuf && !is_device_ptr(sendbuf)) return fail(SFT_E_ARG, "sendbuf must be device memory");
  cudaStream_t s = P->stream;
  const double2* fd = (const double2*)f;
  if (!is_device_ptr(f)) {
    if (!P->f_stage) {
      P->f_stage_bytes = P->nk * sizeof(double2);
      CKR(block_alloc((void**)&P->f_stage, P->f_stage_bytes, s));
    }
    CKR(cudaMemcpyAsync(P->f_stage, f, P->nk * sizeof(double2), cudaMemcpyHostToDevice, s));
    CKR(f_copy_mark(P));
    fd = P->f_stage;
  }
  const int rc = phase1_run(P, fd, (double2*)sendbuf);
  if (fd == P->f_stage) f_copy_wait(P);  // the caller may reuse f once we return
  return rc;
}

extern "C" int sft_apply_phase2(sft_plan_t P, const void* recvbuf, void* u) {
  if (!P || !recvbuf || !u) return fail(SFT_E_ARG, "NULL argument");
  if (!P->sharded) return fail(SFT_E_STATE, "plan is not multi-rank");
  if (!is_device_ptr(recvbuf)) return fail(SFT_E_ARG, "recvbuf must be device memory");
  cudaStream_t s = P->stream;
  const bool u_host = !is_device_ptr(u);
  double2* ud = (double2*)u;
  if (u_host) {
    if (!P->u_stage) {
      P->u_stage_bytes = P->nx * sizeof(double2);
      CKR(block_alloc((void**)&P->u_stage, P->u_stage_bytes, s));
    }
    ud = P->u_stage;
  }
  if (int rc = phase2_run(P, (const double2*)recvbuf, ud, false)) return rc;
  if (u_host) {
    CKR(cudaMemcpyAsync(u, ud, P->nx * sizeof(double2), cudaMemcpyDeviceToHost, s));
    CKR(cudaStreamSynchronize(s));
  }
  return SFT_OK;
}

// ---------------------------------------------------------------------------
// stats / timing
// ---------------------------------------------------------------------------
extern "C" int sft_plan_stats(sft_plan_t P, int64_t* counts_x, int64_t* counts_k, int64_t* pairs, double* info) {
  if (!P) return fail(SFT_E_ARG, "NULL plan");
  const int L = P->L;
  const int64_t PD = ipow64(P->p, P->d);
  double groups = 0, bytes = 0;
  for (int l = 0; l <= L; ++l) {
    if (counts_x) counts_x[l] = P->X.counts[l];
    if (counts_k) counts_k[l] = P->K.counts[l];
    if (pairs) pairs[l] = P->K.counts[l] * P->X.counts[L - l];
  }
  for (int t = 0; t < L; ++t) {
    groups += (double)P->K.counts[t] * P->X.counts[L - t - 1];
    bytes += (P->prec == 1 ? 8.0 : 16.0) * PD *
             ((double)P->K.counts[t] * P->X.counts[L - t] + (double)P->K.counts[t + 1] * P->X.counts[L - t - 1]);
  }
  if (info) {
    info[0] = L;
    info[1] = (double)PD;
    info[2] = (double)P->nx;
    info[3] = (double)P->nk;
    info[4] = 2.0 * P->buf_elems * (P->prec == 1 ? sizeof(float2) : sizeof(double2));
    if (P->plan_ms < 0 && P->plan_ev[1]) {
      float ms = 0;
      cudaEventSynchronize(P->plan_ev[1]);
      cudaEventElapsedTime(&ms, P->plan_ev[0], P->plan_ev[1]);
      P->plan_ms = ms;
    }
    info[5] = P->plan_ms;
    info[6] = groups;
    info[7] = bytes;
  }
  return SFT_OK;
}

extern "C" int sft_set_peer_buffers(sft_plan_t P, void* const* recv) {
  if (!P) return fail(SFT_E_ARG, "NULL plan");
  if (!P->sharded) return fail(SFT_E_STATE, "plan is not multi-rank");
  if (P->world > kMaxPeers) return fail(SFT_E_ARG, "too many ranks for the fused exchange");
  if (!recv) {
    P->peer.clear();
    return SFT_OK;
  }
  P->peer.assign(P->world, nullptr);
  for (int q = 0; q < P->world; ++q) {
    if (!recv[q]) return fail(SFT_E_ARG, "NULL peer buffer");
    P->peer[q] = (double2*)recv[q];
  }
  return SFT_OK;
}

extern "C" int sft_peer_offsets(sft_plan_t P, int64_t* off) {
  if (!P || !off) return fail(SFT_E_ARG, "NULL argument");
  if (!P->sharded) return fail(SFT_E_STATE, "plan is not multi-rank");
  for (int q = 0; q < P->world; ++q) off[q] = P->peer_off[q];
  return SFT_OK;
}

extern "C" int sft_device_alloc(int64_t bytes, void** out) {
  if (!out || bytes < 0) return fail(SFT_E_ARG, "bad arguments");
  CKR(cudaMalloc(out, bytes > 0 ? (size_t)bytes : 1));
  return SFT_OK;
}

extern "C" int sft_device_free(void* p) {
  if (p) CKR(cudaFree(p));
  return SFT_OK;
}

extern "C" int sft_ipc_handle(void* p, void* handle64) {
  if (!p || !handle64) return fail(SFT_E_ARG, "NULL argument");
  cudaIpcMemHandle_t h;
  CKR(cudaIpcGetMemHandle(&h, p));
  std::memcpy(handle64, &h, sizeof(h));
  return SFT_OK;
}

extern "C" int sft_ipc_open(const void* handle64, void** out) {
  if (!handle64 || !out) return fail(SFT_E_ARG, "NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, sizeof(h));
  CKR(cudaIpcOpenMemHandle(out, h, cudaIpcMemLazyEnablePeerAccess));
  return SFT_OK;
}

extern "C" int sft_ipc_close(void* p) {
  if (p) CKR(cudaIpcCloseMemHandle(p));
  return SFT_OK;
}

extern "C" int sft_schedule_bytes(sft_plan_t P, int t, int64_t* bytes, void* dst) {
  if (!P || !bytes || t < 0 || t >= P->L) return fail(SFT_E_ARG, "bad arguments");
  const size_t n = P->sched ? P->sched_off[t + 1] - P->sched_off[t] : 0;
  *bytes = (int64_t)n;
  if (dst && n) {
    CKR(cudaMemcpyAsync(dst, P->sched + P->sched_off[t], n, cudaMemcpyDeviceToHost, P->stream));
    CKR(cudaStreamSynchronize(P->stream));
  }
  return SFT_OK;
}

extern "C" int sft_plan_work(sft_plan_t P, double* w) {
  if (!P || !w) return fail(SFT_E_ARG, "NULL argument");
  const int L = P->L;
  const int64_t PD = ipow64(P->p, P->d);
  double groups = 0, bytes = 0, pairs = 0;
  for (int t = 0; t < L; ++t) {
    groups += (double)P->K.counts[t] * P->X.counts[L - t - 1];
    bytes += (P->prec == 1 ? 8.0 : 16.0) * PD *
             ((double)P->K.counts[t] * P->X.counts[L - t] + (double)P->K.counts[t + 1] * P->X.counts[L - t - 1]);
  }
  for (int t = 0; t <= L; ++t) pairs += (double)P->K.counts[t] * P->X.counts[L - t];
  double acc[3] = {0, 0, 0};
  if (P->sched) {
    std::vector<unsigned char> h;
    if (P->sched_ready) CKR(cudaStreamWaitEvent(P->stream, P->sched_ready, 0));
    for (int t = 0; t < L; ++t) {
      const size_t n = P->sched_off[t + 1] - P->sched_off[t];
      if (!n) continue;
      h.resize(n);
      CKR(cudaMemcpyAsync(h.data(), P->sched + P->sched_off[t], n, cudaMemcpyDeviceToHost, P->stream));
      CKR(cudaStreamSynchronize(P->stream));
      schedule_work(P, h.data(), n, acc);
    }
  }
  w[0] = bytes;
  w[1] = acc[2];
  w[2] = acc[0];
  w[3] = acc[1];
  w[4] = groups;
  w[5] = pairs;
  return SFT_OK;
}

extern "C" int sft_translation_launches(sft_plan_t P, int* n, int* out_level, int* two_level) {
  if (!P || !n) return fail(SFT_E_ARG, "NULL argument");
  const int nl = (int)P->launch_t.size();
  if (P->sharded) {  // multi-rank: one launch per level, split over the two phases
    *n = P->L;
    for (int i = 0; i < P->L; ++i) {
      if (out_level) out_level[i] = P->L - 1 - i;
      if (two_level) two_level[i] = 0;
    }
    return SFT_OK;
  }
  *n = nl;
  for (int i = 0; i < nl; ++i) {
    if (out_level) out_level[i] = P->launch_t[i];
    if (two_level) two_level[i] = P->launch_f2_out[P->launch_t[i]];
  }
  return SFT_OK;
}

extern "C" int sft_set_timing(sft_plan_t P, int enable) {
  if (!P) return fail(SFT_E_ARG, "NULL plan");
  if (enable < 0 || enable > 2) return fail(SFT_E_ARG, "timing mode must be 0, 1 or 2");
  P->timing = enable;
  return SFT_OK;
}

extern "C" int sft_last_timing(sft_plan_t P, double* t_ms, double* per_level_ms) {
  if (!P) return fail(SFT_E_ARG, "NULL plan");
  if (t_ms)
    for (int i = 0; i < 4; ++i) t_ms[i] = P->last_ms[i];
  if (per_level_ms)
    for (int t = 0; t < P->L; ++t) per_level_ms[t] = t < (int)P->level_ms.size() ? P->level_ms[t] : 0.0;
  return SFT_OK;
}
