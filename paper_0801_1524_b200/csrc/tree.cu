// tree.cu -- step 1 of the butterfly: adaptive quadtrees /
// octrees T_X and T_K with unit-width leaves, keeping only non-empty boxes.
//
// GPU build, one pass per tree:
//   1. leaf Morton key per point (c = min(floor(y), N-1) per axis; axis 0 is
//      the most significant bit of each d-bit digit), domain check;
//   2. radix sort of (key, index) -- CUB, compiled into this library;
//   3. for every point the coarsest level at which it opens a new box
//      (from the highest differing bit with its predecessor), one histogram
//      -> exact box counts per level with a single host sync for both trees;
//   4. per level: flag -> inclusive scan -> box ids; box keys, parent, child
//      begin and child mask (children of a box are contiguous in Morton order).
#include <cub/cub.cuh>

#include "sft_internal.cuh"

namespace sft {

__global__ void k_leaf_keys(const double* __restrict__ pts, int64_t n, int d, int L, double Nf, int64_t N,
                            uint64_t* __restrict__ key, int32_t* __restrict__ idx, int* err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint64_t c[kMaxDim] = {0, 0, 0};
  for (int a = 0; a < d; ++a) {
    double y = pts[i * d + a];
    if (!(y >= 0.0 && y <= Nf)) {  // also catches NaN
      atomicOr(err, 1);
      y = 0.0;
    }
    int64_t ci = (int64_t)floor(y);
    if (ci > N - 1) ci = N - 1;
    c[a] = (uint64_t)ci;
  }
  uint64_t k = 0;
  for (int b = L - 1; b >= 0; --b)
    for (int a = 0; a < d; ++a) k = (k << 1) | ((c[a] >> b) & 1ull);
  key[i] = k;
  idx[i] = (int32_t)i;
}

// coarsest level at which sorted point i starts a new box
__global__ void k_min_level(const uint64_t* __restrict__ key, int64_t n, int d, int L, uint8_t* __restrict__ ml,
                            unsigned long long* __restrict__ hist) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lev = 0;
  if (i > 0) {
    uint64_t x = key[i] ^ key[i - 1];
    if (x == 0) {
      lev = L + 1;  // same leaf: never opens a box
    } else {
      int hb = 63 - __clzll((long long)x);
      lev = L - hb / d;
    }
  }
  ml[i] = (uint8_t)lev;
  if (lev <= L) atomicAdd(&hist[lev], 1ull);
}

__global__ void k_flags(const uint8_t* __restrict__ ml, int64_t n, int lev, int32_t* __restrict__ flag) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) flag[i] = ml[i] <= lev ? 1 : 0;
}

// bid: inclusive scan of flags at this level (box id + 1 of every point)
// bid_up: same for level lev+1 (nullptr at the leaf level)
__global__ void k_fill_level(const uint64_t* __restrict__ key, const uint8_t* __restrict__ ml, int64_t n, int d,
                             int L, int lev, const int32_t* __restrict__ bid, const int32_t* __restrict__ bid_up,
                             uint64_t* __restrict__ bkey, int32_t* __restrict__ child_begin,
                             uint32_t* __restrict__ child_mask, int32_t* __restrict__ parent_up,
                             int32_t* __restrict__ first_pt) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int m = ml[i];
  int32_t b = bid[i] - 1;
  if (m <= lev) {
    bkey[b] = key[i] >> (d * (L - lev));
    if (first_pt) first_pt[b] = (int32_t)i;
    if (bid_up) child_begin[b] = bid_up[i] - 1;
  }
  if (bid_up && m <= lev + 1) {
    int32_t c = bid_up[i] - 1;
    parent_up[c] = b;
    uint32_t bits = (uint32_t)((key[i] >> (d * (L - lev - 1))) & ((1u << d) - 1));
    atomicOr(&child_mask[b], 1u << bits);
  }
}

__global__ void k_gather_pts(const double* __restrict__ pts, const int32_t* __restrict__ perm, int64_t n, int d,
                             double* __restrict__ out) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t j = perm[i];
  for (int a = 0; a < d; ++a) out[i * d + a] = pts[j * d + a];
}

__global__ void k_set_i32(int32_t* p, int32_t v) { *p = v; }

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

#define CK(x)                                                   \
  do {                                                          \
    cudaError_t e_ = (x);                                       \
    if (e_ != cudaSuccess) {                                    \
      if (err) *err = std::string(#x) + ": " + cudaGetErrorString(e_); \
      return SFT_E_CUDA;                                        \
    }                                                           \
  } while (0)

template <class T>
static cudaError_t dalloc(T** p, size_t n, cudaStream_t s) {
  return cudaMallocAsync((void**)p, (n > 0 ? n : 1) * sizeof(T), s);
}

struct Scratch {
  uint64_t* keys_in = nullptr;
  int32_t* idx_in = nullptr;
  uint8_t* ml = nullptr;
  int32_t* bidA = nullptr;
  int32_t* bidB = nullptr;
  unsigned long long* hist = nullptr;
  void* cub_tmp = nullptr;
  size_t cub_bytes = 0;
};

static int tree_phase1(sft_plan_s* P, Tree& T, const double* pts, int64_t n, Scratch& S, std::string* err) {
  cudaStream_t s = P->stream;
  const int d = P->d, L = P->L;
  T.d = d;
  T.L = L;
  T.npts = n;
  CK(dalloc(&S.keys_in, n, s));
  CK(dalloc(&S.idx_in, n, s));
  CK(dalloc(&T.keys_sorted, n, s));
  CK(dalloc(&T.perm, n, s));
  CK(dalloc(&S.ml, n, s));
  CK(dalloc(&S.hist, L + 1, s));
  CK(cudaMemsetAsync(S.hist, 0, (L + 1) * sizeof(unsigned long long), s));
  k_leaf_keys<<<nblk(n, 256), 256, 0, s>>>(pts, n, d, L, (double)P->N, P->N, S.keys_in, S.idx_in, P->d_err);
  count_launch();
  CK(cudaGetLastError());
  size_t need = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, need, S.keys_in, T.keys_sorted, S.idx_in, T.perm, (int)n, 0, d * L, s));
  size_t need2 = 0;
  CK(cub::DeviceScan::InclusiveSum(nullptr, need2, (int32_t*)nullptr, (int32_t*)nullptr, (int)n, s));
  S.cub_bytes = need > need2 ? need : need2;
  CK(cudaMallocAsync(&S.cub_tmp, S.cub_bytes > 0 ? S.cub_bytes : 1, s));
  CK(cub::DeviceRadixSort::SortPairs(S.cub_tmp, need, S.keys_in, T.keys_sorted, S.idx_in, T.perm, (int)n, 0, d * L,
                                     s));
  k_min_level<<<nblk(n, 256), 256, 0, s>>>(T.keys_sorted, n, d, L, S.ml, S.hist);
  count_launch();
  CK(cudaGetLastError());
  return SFT_OK;
}

static int tree_phase2(sft_plan_s* P, Tree& T, const double* pts, const std::vector<int64_t>& hist, Scratch& S,
                       std::string* err) {
  cudaStream_t s = P->stream;
  const int d = P->d, L = P->L;
  const int64_t n = T.npts;
  T.lev.assign(L + 1, TreeLevel());
  T.counts.assign(L + 1, 0);
  int64_t acc = 0;
  for (int l = 0; l <= L; ++l) {
    acc += hist[l];
    T.counts[l] = acc;
    T.lev[l].n = acc;
  }
  for (int l = 0; l <= L; ++l) {
    TreeLevel& lv = T.lev[l];
    CK(dalloc(&lv.key, lv.n, s));
    if (l < L) {
      CK(dalloc(&lv.child_begin, lv.n, s));
      CK(dalloc(&lv.child_mask, lv.n, s));
      CK(cudaMemsetAsync(lv.child_mask, 0, lv.n * sizeof(uint32_t), s));
    }
    if (l > 0) CK(dalloc(&lv.parent, lv.n, s));
  }
  CK(dalloc(&T.first_pt, T.lev[L].n + 1, s));
  CK(dalloc(&T.pts_sorted, n * d, s));
  CK(dalloc(&S.bidA, n, s));
  CK(dalloc(&S.bidB, n, s));
  int32_t* bid_up = nullptr;
  int32_t* bufs[2] = {S.bidA, S.bidB};
  for (int l = L; l >= 0; --l) {
    int32_t* bid = bufs[l & 1];
    k_flags<<<nblk(n, 256), 256, 0, s>>>(S.ml, n, l, bid);
    count_launch();
    CK(cudaGetLastError());
    size_t nb = S.cub_bytes;
    CK(cub::DeviceScan::InclusiveSum(S.cub_tmp, nb, bid, bid, (int)n, s));
    TreeLevel& lv = T.lev[l];
    k_fill_level<<<nblk(n, 256), 256, 0, s>>>(T.keys_sorted, S.ml, n, d, L, l, bid, bid_up, lv.key, lv.child_begin,
                                              lv.child_mask, l < L ? T.lev[l + 1].parent : nullptr,
                                              l == L ? T.first_pt : nullptr);
    count_launch();
    CK(cudaGetLastError());
    bid_up = bid;
  }
  k_set_i32<<<1, 1, 0, s>>>(T.first_pt + T.lev[L].n, (int32_t)n);
  k_gather_pts<<<nblk(n, 256), 256, 0, s>>>(pts, T.perm, n, d, T.pts_sorted);
  count_launch(2);
  CK(cudaGetLastError());
  CK(cudaFreeAsync(S.keys_in, s));
  CK(cudaFreeAsync(S.idx_in, s));
  CK(cudaFreeAsync(S.ml, s));
  CK(cudaFreeAsync(S.hist, s));
  CK(cudaFreeAsync(S.bidA, s));
  CK(cudaFreeAsync(S.bidB, s));
  CK(cudaFreeAsync(S.cub_tmp, s));
  return SFT_OK;
}

int build_trees(sft_plan_s* P, const double* x_dev, const double* k_dev, std::string* err) {
  Scratch SX, SK;
  int rc = tree_phase1(P, P->X, x_dev, P->nx, SX, err);
  if (rc) return rc;
  rc = tree_phase1(P, P->K, k_dev, P->nk, SK, err);
  if (rc) return rc;
  // one host sync for both trees: level histograms + domain error flag
  const int L = P->L;
  std::vector<unsigned long long> h(2 * (L + 1) + 1);
  CK(cudaMemcpyAsync(h.data(), SX.hist, (L + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost, P->stream));
  CK(cudaMemcpyAsync(h.data() + L + 1, SK.hist, (L + 1) * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                     P->stream));
  int herr = 0;
  CK(cudaMemcpyAsync(&herr, P->d_err, sizeof(int), cudaMemcpyDeviceToHost, P->stream));
  CK(cudaStreamSynchronize(P->stream));
  if (herr) {
    if (err) *err = "a coordinate is non-finite or outside [0,N]";
    // release scratch before failing
    cudaFreeAsync(SX.keys_in, P->stream); cudaFreeAsync(SX.idx_in, P->stream); cudaFreeAsync(SX.ml, P->stream);
    cudaFreeAsync(SX.hist, P->stream); cudaFreeAsync(SX.cub_tmp, P->stream);
    cudaFreeAsync(SK.keys_in, P->stream); cudaFreeAsync(SK.idx_in, P->stream); cudaFreeAsync(SK.ml, P->stream);
    cudaFreeAsync(SK.hist, P->stream); cudaFreeAsync(SK.cub_tmp, P->stream);
    return SFT_E_DOMAIN;
  }
  std::vector<int64_t> hx(L + 1), hk(L + 1);
  for (int l = 0; l <= L; ++l) {
    hx[l] = (int64_t)h[l];
    hk[l] = (int64_t)h[L + 1 + l];
  }
  rc = tree_phase2(P, P->X, x_dev, hx, SX, err);
  if (rc) return rc;
  return tree_phase2(P, P->K, k_dev, hk, SK, err);
}

void free_tree(Tree& T, cudaStream_t s) {
  for (auto& lv : T.lev) {
    if (lv.key) cudaFreeAsync(lv.key, s);
    if (lv.child_begin) cudaFreeAsync(lv.child_begin, s);
    if (lv.child_mask) cudaFreeAsync(lv.child_mask, s);
    if (lv.parent) cudaFreeAsync(lv.parent, s);
  }
  T.lev.clear();
  if (T.first_pt) cudaFreeAsync(T.first_pt, s);
  if (T.perm) cudaFreeAsync(T.perm, s);
  if (T.pts_sorted) cudaFreeAsync(T.pts_sorted, s);
  if (T.keys_sorted) cudaFreeAsync(T.keys_sorted, s);
  T.first_pt = nullptr;
  T.perm = nullptr;
  T.pts_sorted = nullptr;
  T.keys_sorted = nullptr;
}

}  // namespace sft
