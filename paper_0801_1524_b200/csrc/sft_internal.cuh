// sft_internal.cuh -- internal structures of libsft (B200 butterfly SFT).
// Nothing here is shared with oracle/ (test infrastructure).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/sft.h"

namespace sft {

// Box-relative formulation (derived from eq. M1/E1):
//   g^{AB} = M12 f^{AB} per axis, (M12)_l = e^{2 pi i a l/(p-1)} (a = index of A),
//   stored as h^{AB} = (x)_axes diag(e^{i pi m/(p-1)}) g^{AB}  ("h-representation"):
//   leaf:   h^{A0 B}_m = sum_{k_j in B} f_j e^{i pi sum_ax s_ax} prod_ax r_{m_ax}(s_ax),
//           s = k_j - c^B, r_m(s) = invD_m prod_{q != m} sin(pi (s (p-1) - q)/(p-1)^2)  (real)
//   level:  h^{AB} = sum_{present B_c} (x)_ax T[alpha_ax][beta_ax] h^{A' B_c},
//           T[alpha][beta] = c_ab (RC_beta + i (2 alpha - 1) RS_beta), RC/RS real p x p
//   final:  u(x) = sum_l prod_ax e^{i pi l_ax (2 xi_ax - 1)/(p-1)} h^{A B0}_l, xi = x - c^A
// The tables depend on p only; they are built on the host in long double from
// the Lagrange / sine-product closed forms (tables.cpp); no G^{-1} anywhere.

constexpr int kMaxDim = 3;
constexpr int kMaxLevels = 21;  // N <= 2^20
constexpr int kMaxPeers = 8;    // ranks of the fused (peer-store) exchange

struct TreeLevel {
  int64_t n = 0;                  // non-empty boxes at this level
  uint64_t* key = nullptr;        // [n] Morton key of each box (sorted)
  int32_t* child_begin = nullptr; // [n] first child at level+1 (level < L)
  uint32_t* child_mask = nullptr; // [n] bit c set <=> child c present (level < L)
  int32_t* parent = nullptr;      // [n] parent index at level-1 (level > 0)
};

struct Tree {
  int d = 0, L = 0;
  int64_t npts = 0;
  std::vector<TreeLevel> lev;      // [L+1]
  std::vector<int64_t> counts;     // host copy of lev[l].n
  int32_t* first_pt = nullptr;     // [n_leaf+1] CSR of sorted points per leaf
  int32_t* leaf_of = nullptr;      // [npts] leaf index of each sorted point
  int32_t* perm = nullptr;         // [npts] sorted position -> user index
  double* pts_sorted = nullptr;    // [npts][d]
  void* arena = nullptr;           // one allocation holding every array above (X owns both trees')
  size_t arena_bytes = 0;
};

struct DeviceTables {
  int p = 0;
  double2* V = nullptr;       // [2][2][p][p]  V[alpha][beta][m][l']
  double* leaf_invD = nullptr;  // [p]  1 / prod_{q != m} sin(pi (m-q)/(p-1)^2)
};

// Host-side long double construction (tables.cpp).
void build_tables_host(int p, std::vector<double>& V /* 2*4*p*p */, std::vector<double>& invD /* p */,
                       std::vector<double>* RC = nullptr /* 2*p*p */, std::vector<double>* RS = nullptr);
const DeviceTables* get_device_tables(int p, std::string* err);

struct Partition {
  int sk = 0, sx = 0, m = 0;
  std::vector<int64_t> k_lo, k_hi;  // [world] box ranges at level sk
  std::vector<int64_t> x_lo, x_hi;  // [world] box ranges at level sx
};

// Range of boxes at level `lev` that descend from boxes [lo, hi) at level `s`.
struct LevelRange {
  int64_t lo = 0, hi = 0;
};

}  // namespace sft

struct sft_plan_s {
  int d = 0, p = 0, L = 0;
  int64_t N = 0, nx = 0, nk = 0;
  int rank = 0, world = 1;
  bool sharded = false;  // the two-phase multi-rank path (world > 1, or forced on one rank)
  int dev = 0;   // CUDA device the plan was created on (its pooled events belong to it)
  int prec = 0;  // 0 = FP64 charges (complex128), 1 = FP32 charges (complex64)
  int conj = 0;  // adjoint plan: conjugate the charges on input and the potentials on output
  int ffmod = 0; // far-field plan (sft_farfield_plan): source (forward) / target (adjoint) modulation e^{-+i pi sum k}
  int pds = 0;   // stride (complex elements) of one pair array in the level buffers
  cudaStream_t stream = nullptr;
  sft::Tree X, K;
  const sft::DeviceTables* tab = nullptr;
  // two live level buffers, complex128 (or complex64 if prec == 1)
  double2* buf[2] = {nullptr, nullptr};
  size_t buf_elems = 0;
  // level buffers of the multi-RHS apply (sft_apply_batch): [bufb_rhs][buf_elems] each, grown on demand
  double2* bufb[2] = {nullptr, nullptr};
  int bufb_rhs = 0;
  int64_t stage_rhs = 0;  // RHS capacity of f_stage / u_stage (host-pointer batches)
  // staging for host pointers
  double2* f_stage = nullptr;
  double2* u_stage = nullptr;
  size_t f_stage_bytes = 0, u_stage_bytes = 0, blk_bytes = 0;  // sizes of the cached blocks (block_free)
  cudaEvent_t f_copied = nullptr;  // recorded after a host f's staging copy (sft_apply waits on it)
  int* d_err = nullptr;
  // multi-GPU
  sft::Partition part;
  std::vector<sft::LevelRange> k_rng;  // [L+1] this rank's T_K range per level (phase 1)
  std::vector<sft::LevelRange> x_rng;  // [L+1] this rank's T_X range per level (phase 2)
  int64_t x_pt_lo = 0, x_pt_hi = 0;     // sorted target range of this rank's T_X leaves
  int64_t k_src_lo = 0, k_src_hi = 0;   // sorted source range of this rank's T_K leaves
  std::vector<int64_t> send_counts, recv_counts;  // [world] complex elements
  int64_t* d_seg = nullptr;  // device [2*world+1]: a-boundaries at level L-m, send segment bases
  std::vector<int64_t> seg_host;   // host copy of the same
  std::vector<int64_t> peer_off;   // [world] element offset of this rank's segment in each receiver's buffer
  std::vector<double2*> peer;      // [world] receive buffers (fused exchange), empty = use the send buffer
  // in-library collectives (opts.nccl_id): communicator (cached per id, not owned),
  // exchange buffers, and the u all-gather: rank q's targets are the sorted
  // points [u_bounds[q], u_bounds[q+1]), gathered as [world][u_cnt]
  void* comm = nullptr;
  double2* xsend = nullptr;
  double2* xrecv = nullptr;
  double2* u_all = nullptr;
  int64_t* d_ubounds = nullptr;
  int64_t u_cnt = 0;
  std::vector<int64_t> u_bounds;
  // translation launches of a world-1 apply: output level and whether it is a
  // two-level launch (levels t+1, t from t+2); schedules per launch
  std::vector<int> launch_t, launch_f2_out;  // launch order (output levels); f2 flag per output level
  // tile schedules of the translation launches (one allocation; offsets per launch,
  // for multi-rank plans per level t)
  unsigned char* sched = nullptr;
  int* tctr = nullptr;  // [L][2] dynamic tile-scheduling counters per translation launch (after the schedules)
  std::vector<size_t> sched_off;
  cudaEvent_t sched_fork = nullptr, sched_ready = nullptr;  // schedule kernel on the side stream
  cudaEvent_t sched_first = nullptr;  // the first translation launch's schedule (world 1)
  // timing
  int timing = 0;  // sft_set_timing: 0 off, 1 events around every launch, 2 around the translation chain
  cudaEvent_t ev[64];
  int n_ev = 0;
  int ev_created = 0;
  double last_ms[4] = {0, 0, 0, 0};
  std::vector<double> level_ms;
  double plan_ms = 0;               // device time of sft_plan (events below), read lazily
  cudaEvent_t plan_ev[2] = {nullptr, nullptr};
};

namespace sft {

// api.cu: device blocks of destroyed plans reused by the next plans (per device)
cudaError_t block_alloc(void** out, size_t bytes, cudaStream_t s);
void block_free(void* p, size_t bytes, cudaStream_t s);

// tree.cu
int build_trees(sft_plan_s* P, const double* x_dev, const double* k_dev, std::string* err);
void free_tree(Tree& T, cudaStream_t s);

// kernels.cu
struct LevelDims {
  // translation from level t+1 (input) to level t (output)
  int t;
  const int32_t* cbK;  // T_K level t child_begin
  const uint32_t* mK;  // T_K level t child_mask
  const int32_t* cbX;  // T_X level L-t-1 child_begin
  const uint32_t* mX;  // T_X level L-t-1 child_mask
  int64_t b_lo, b_hi;   // B range at level t (groups)
  int64_t ap_lo, ap_hi; // A' range at level L-t-1 (groups)
  int64_t in_b0, in_nA, in_a0;   // input layout: [(iBc - in_b0) * in_nA + (iA' - in_a0)]
  int64_t out_b0, out_nA, out_a0; // output layout: [(iB - out_b0) * out_nA + (iA - out_a0)]
  const int64_t* seg;  // exchange mapping (nullptr = plain layout), see api.cu
  int nseg;
  const unsigned char* sched = nullptr;  // tile schedule of this level (translate.cu, built by sft_plan)
  // fused exchange: outputs of send-layout pair index i in segment q go to
  // peer[q] + peer_off[q] + (i - peer_seg[q]) * p^d
  int npeer = 0;
  double2* peer[kMaxPeers] = {};
  int64_t peer_off[kMaxPeers] = {};
  int64_t peer_seg[kMaxPeers + 1] = {};
  // two-level (radix-4) launch, 2D: levels t+1 and t from level t+2 in one
  // pass over super-groups (A'', B); see translate.cu schedule_f2
  int f2 = 0;
  const int32_t* cbK1 = nullptr;  // T_K level t+1
  const uint32_t* mK1 = nullptr;
  const int32_t* cbX2 = nullptr;  // T_X level L-t-2 (A'' range in ap_lo/ap_hi)
  const uint32_t* mX2 = nullptr;
  // multi-RHS batch (sft_apply_batch): nrhs independent charge vectors through
  // the same schedule; RHS r of the input / output level lives at in/out + r * rs
  // (elements of the stored type)
  int nrhs = 1;
  int64_t rs = 0;
  // dynamic tile scheduling counters of this launch ([next item, CTAs done];
  // zeroed by the plan's schedule kernel, reset by the launch's last CTA), or
  // nullptr for the static grid-stride assignment
  int* ctr = nullptr;
};

// level buffers are void*: complex128 (prec 0) or complex64 (prec 1) pair arrays of stride P->pds
// nrhs > 1: charge vector r at f + r * ldf (complex128), its leaf level at out + r * ors (stored elements)
cudaError_t launch_leaf(const sft_plan_s* P, const double2* f, void* out, int64_t b_lo, int64_t b_hi, int nrhs = 1,
                        int64_t ldf = 0, int64_t ors = 0);
cudaError_t launch_translate(const sft_plan_s* P, const LevelDims& L, const void* in, void* out);
// two-level launches available for this plan (2D FP64 single-GPU; SFT_F2=0 disables)
bool two_level_supported(const sft_plan_s* P);
// work of one translation launch from a host copy of its tile schedule:
// out[0] += super-tiles, out[1] += fiber tasks, out[2] += executed FP64 flops
void schedule_work(const sft_plan_s* P, const unsigned char* h, size_t bytes, double* out);
// tile schedule of one level (sizes and builder; 0 bytes when the kernel needs none)
size_t schedule_bytes(const sft_plan_s* P, const LevelDims& L);
// builds the schedules of nlev levels (dims L[i], destination dst[i]) in one launch
cudaError_t launch_schedule(const sft_plan_s* P, const LevelDims* L, int nlev, unsigned char* const* dst,
                            cudaStream_t st);
// debug: validate a level's schedule against its input/output pair counts (sets *err bit 2)
cudaError_t check_schedule(const sft_plan_s* P, const LevelDims& L, const unsigned char* sched, int64_t in_pairs,
                           int64_t out_pairs, int* err);
// step 4 for the sorted targets [i_lo, i_hi) (the points of leaves a_lo...); g0 holds leaves from a_lo on
// nrhs > 1: level-0 charges of RHS r at g0 + r * hrs (stored elements), potentials at u + r * ldu
// sorted_out: u[j - i_lo] for sorted target j (the all-gather layout) instead of u[perm[j]]
cudaError_t launch_final(const sft_plan_s* P, const void* g0, double2* u, int64_t a_lo, int64_t i_lo, int64_t i_hi,
                         int nrhs = 1, int64_t hrs = 0, int64_t ldu = 0, bool sorted_out = false);
// u[perm[j]] = u_all[q * cnt + j - bounds[q]] for the rank q with bounds[q] <= j < bounds[q+1]
cudaError_t launch_unsort(const double2* u_all, int64_t cnt, const int64_t* bounds, int world, const int32_t* perm,
                          double2* u, int64_t n, cudaStream_t s);

// comm.cu: NCCL (dlopen'ed; SFT_E_NCCL on failure, message in *err)
int nccl_comm_get(const void* id128, int rank, int world, void** comm, std::string* err);
int nccl_exchange(void* comm, const double2* send, const int64_t* send_counts, double2* recv,
                  const int64_t* recv_counts, int world, cudaStream_t s, std::string* err);
int nccl_allgather(void* comm, const double2* send, double2* recv, int64_t count, cudaStream_t s, std::string* err);
cudaError_t launch_zero(double2* p, int64_t n, cudaStream_t s);
// far-field adapter: x = N/2 - kappa xhat/(2 pi), k = N y (device arrays [n][d])
cudaError_t launch_ff_coords(const double* xhat, int64_t nx, const double* y, int64_t ny, int d, double kappa,
                             int64_t N, double* x, double* k, cudaStream_t s);

template <int B, int E>
struct Pow {
  static constexpr int v = B * Pow<B, E - 1>::v;
};
template <int B>
struct Pow<B, 0> {
  static constexpr int v = 1;
};

// Stride (elements) of one pair array in the level buffers and stages: p^d,
// rounded up to even for FP32 (16-byte bulk copies) and -- SFT_PAD_EVEN -- for
// FP64 too (every array starts on a 32-byte sector: no sector is shared by two
// arrays written by different CTAs)
#ifndef SFT_PAD_EVEN
#define SFT_PAD_EVEN 0
#endif
template <typename E, int PD>
struct StrideT {
  static constexpr int v = (sizeof(E) == 8 || SFT_PAD_EVEN) ? PD + (PD & 1) : PD;
};
inline int pair_stride(int pd, int prec) { return (prec == 1 || SFT_PAD_EVEN) ? pd + (pd & 1) : pd; }

#define SFT_DISPATCH(D_, P_, CALL)                                       \
  do {                                                                   \
    if (D_ == 2 && P_ == 5) { constexpr int D = 2, P = 5; CALL; }        \
    else if (D_ == 2 && P_ == 7) { constexpr int D = 2, P = 7; CALL; }   \
    else if (D_ == 2 && P_ == 9) { constexpr int D = 2, P = 9; CALL; }   \
    else if (D_ == 3 && P_ == 5) { constexpr int D = 3, P = 5; CALL; }   \
    else if (D_ == 3 && P_ == 7) { constexpr int D = 3, P = 7; CALL; }   \
    else if (D_ == 3 && P_ == 9) { constexpr int D = 3, P = 9; CALL; }   \
    else return cudaErrorInvalidValue;                                   \
  } while (0)

// Per-device cache of a value computed once per CUDA device (launch attributes,
// occupancy grids, device tables): a process may plan on several GPUs, so
// nothing derived from one device may be reused on another.
template <typename T>
struct PerDevice {
  static constexpr int kMaxDev = 64;
  std::mutex mu;
  T val[kMaxDev] = {};
  bool ok[kMaxDev] = {};
  // *out = the cached value of the current device, computing it with
  // init(dev, &value) (returns cudaError_t) on first use
  template <class F>
  cudaError_t get(T* out, F init) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= kMaxDev) return cudaErrorInvalidDevice;
    std::lock_guard<std::mutex> lk(mu);
    if (!ok[dev]) {
      T v{};
      e = init(dev, &v);
      if (e != cudaSuccess) return e;
      val[dev] = v;
      ok[dev] = true;
    }
    *out = val[dev];
    return cudaSuccess;
  }
};

// SFT_PLAN_TRACE=1: host-time milestones of sft_plan (api.cu)
void trace_mark(const char* what, cudaStream_t s = nullptr, bool dev = false);  // dev: also a device event on s

// number of kernels this library has launched (own kernels; CUB's internal
// sort/scan kernels are not counted), for bench.py's gpu_launches
void count_launch(int n = 1);

// SFT_PDL=0 disables programmatic dependent launch (ablation)
inline bool pdl_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SFT_PDL");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// Launch with programmatic stream serialization (PDL): the kernel may start
// while the previous kernel on the stream drains; it must execute
// griddepcontrol.wait before touching that kernel's data (or anything an
// earlier kernel wrote), and every kernel triggers its own dependents
// (griddepcontrol.launch_dependents) only after that wait, so a dependent's
// pre-wait prologue never overlaps anything but its direct predecessor.
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t st,
                       Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}


}  // namespace sft
