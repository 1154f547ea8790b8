// tree.cu -- step 1 of the butterfly: adaptive quadtrees /
// octrees T_X and T_K with unit-width leaves, keeping only non-empty boxes.
//
// Both trees are built together, in four launches and one host sync:
//   1. k_leaf_keys: leaf Morton key of every point of x and k (c = min(floor(y),
//      N-1) per axis; axis 0 is the most significant bit of each d-bit digit),
//      tagged with a tree bit above the d*L key bits (X first), domain check;
//   2. one radix sort of (key, index) over d*L+1 bits -- CUB, compiled into
//      this library;
//   3. k_count: per sorted point the coarsest level at which it opens a new
//      box (highest differing key bit with its predecessor; the first point of
//      each tree opens the root), and per 1024-point block the number of
//      box-opening points at every level (warp ballots, no global atomics);
//   4. k_fill: per block, the exclusive prefix of those counts over the
//      earlier blocks of the same tree, then for every point its box id at
//      every level (inclusive count of openers - 1); box-opening points write
//      the box's key, parent, first child and their bit in the parent's child
//      mask; every point writes its sorted coordinates and permutation entry;
//      the last block of each tree writes the per-level box counts.
// Level arrays live in one arena sized by the upper bound min(n, 2^(d*l)) per
// level, so nothing on the device waits for the host; the single sync at the
// end reads the exact counts (the apply needs them to size grids and buffers).
#include <atomic>
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "sft_internal.cuh"

namespace sft {

constexpr int kBlk = 1024;  // points per block in k_count / k_fill

__device__ __forceinline__ uint64_t spread2(uint64_t x) {  // bit b -> bit 2b
  x &= 0xFFFFFFFFull;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}
__device__ __forceinline__ uint64_t spread3(uint64_t x) {  // bit b -> bit 3b (b < 21)
  x &= 0x1FFFFFull;
  x = (x | (x << 32)) & 0x1F00000000FFFFull;
  x = (x | (x << 16)) & 0x1F0000FF0000FFull;
  x = (x | (x << 8)) & 0x100F00F00F00F00Full;
  x = (x | (x << 4)) & 0x10C30C30C30C30C3ull;
  x = (x | (x << 2)) & 0x1249249249249249ull;
  return x;
}

template <typename KT>
__global__ void k_leaf_keys(const double* __restrict__ x, int64_t nx, const double* __restrict__ k, int64_t nk,
                            int d, int L, double Nf, int64_t N, KT* __restrict__ key,
                            int32_t* __restrict__ idx, int* err) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= nx + nk) return;
  const bool tk = i >= nx;
  const double* pts = tk ? k + (i - nx) * d : x + i * d;
  uint64_t c[kMaxDim] = {0, 0, 0};
  for (int a = 0; a < d; ++a) {
    double y = pts[a];
    if (!(y >= 0.0 && y <= Nf)) {  // also catches NaN
      atomicOr(err, 1);
      y = 0.0;
    }
    int64_t ci = (int64_t)floor(y);
    if (ci > N - 1) ci = N - 1;
    c[a] = (uint64_t)ci;
  }
  // Morton interleave, axis 0 the most significant bit of each d-bit digit, tree
  // bit above the d*L key bits (bit spreading by magic masks; c < 2^20)
  uint64_t kk;
  if (d == 2) {
    kk = (spread2(c[0]) << 1) | spread2(c[1]);
  } else {
    kk = (spread3(c[0]) << 2) | (spread3(c[1]) << 1) | spread3(c[2]);
  }
  kk |= (tk ? 1ull : 0ull) << (d * L);
  key[i] = (KT)kk;
  idx[i] = (int32_t)i;
}

// Small trees (<= kBlockSortMax points each): both trees sorted in one launch,
// one 1024-thread block per tree with a block-wide radix sort in shared memory
// (cub::BlockRadixSort: stable, so ties keep the input = index order exactly as
// the device-wide sort).  Keys are compared on bits [0, bits); padding items
// carry all-ones keys and sort behind every real item (stable).
#ifndef SFT_BS_BITS
#define SFT_BS_BITS 4  // radix digit bits of the block sort
#endif
// Items per thread: the smallest instantiation that holds the larger tree
// (padding items cost a full sort pass each: C1's 10K-point trees take 11 items
// per thread instead of 16, C0's 643 points 1).
constexpr int kBlockSortItems = 16;
constexpr int kBlockSortMax = 1024 * kBlockSortItems;
template <typename KT, int ITEMS>
__global__ __launch_bounds__(1024) void k_block_sort(const KT* __restrict__ kin, const int32_t* __restrict__ iin,
                                                     KT* __restrict__ kout, int32_t* __restrict__ iout, int64_t nx,
                                                     int64_t nk, int bits) {
  constexpr int kBlockSortItems = ITEMS;
  using BRS = cub::BlockRadixSort<KT, 1024, kBlockSortItems, int32_t, SFT_BS_BITS>;
  extern __shared__ __align__(16) unsigned char bs_smem[];
  auto& tmp = *reinterpret_cast<typename BRS::TempStorage*>(bs_smem);
  const int64_t lo = blockIdx.x == 0 ? 0 : nx;
  const int64_t n = blockIdx.x == 0 ? nx : nk;
  KT k[kBlockSortItems];
  int32_t v[kBlockSortItems];
#pragma unroll
  for (int i = 0; i < kBlockSortItems; ++i) {
    const int64_t idx = (int64_t)threadIdx.x * kBlockSortItems + i;
    k[i] = idx < n ? kin[lo + idx] : ~(KT)0;
    v[i] = idx < n ? iin[lo + idx] : INT32_MAX;
  }
  BRS(tmp).SortBlockedToStriped(k, v, 0, bits);
#pragma unroll
  for (int i = 0; i < kBlockSortItems; ++i) {
    const int64_t pos = (int64_t)i * 1024 + threadIdx.x;
    if (pos < n) {
      kout[lo + pos] = k[i];
      iout[lo + pos] = v[i];
    }
  }
}

struct BlockMap {
  int64_t nx, n;
  int nbx;  // blocks covering [0, nx); blocks >= nbx cover [nx, n)
  __device__ __forceinline__ void get(int b, int& tree, int64_t& ts, int64_t& lo, int64_t& hi) const {
    tree = b >= nbx;
    ts = tree ? nx : 0;
    lo = ts + (int64_t)(tree ? b - nbx : b) * kBlk;
    hi = min(lo + kBlk, tree ? n : nx);
  }
};

// level at which sorted point i (of the tree starting at ts) opens a box;
// L+1 = never (same leaf as its predecessor)
template <typename KT>
__device__ __forceinline__ int open_level(const KT* key, int64_t i, int64_t ts, int d, int L) {
  if (i == ts) return 0;
  const uint64_t x = (uint64_t)key[i] ^ (uint64_t)key[i - 1];
  if (x == 0) return L + 1;
  const int hb = 63 - __clzll((long long)x);
  return L - hb / d;
}

template <typename KT>
__global__ __launch_bounds__(kBlk) void k_count(const KT* __restrict__ key, BlockMap bm, int d, int L,
                                                uint8_t* __restrict__ ml, int32_t* __restrict__ counts) {
  __shared__ int cnt[kMaxLevels];
  int tree;
  int64_t ts, lo, hi;
  bm.get(blockIdx.x, tree, ts, lo, hi);
  if (threadIdx.x <= L) cnt[threadIdx.x] = 0;
  __syncthreads();
  const int64_t i = lo + threadIdx.x;
  int m = L + 1;
  if (i < hi) {
    m = open_level(key, i, ts, d, L);
    ml[i] = (uint8_t)m;
  }
  const int lane = threadIdx.x & 31;
  for (int l = 0; l <= L; ++l) {
    const unsigned b = __ballot_sync(0xffffffffu, m <= l);
    if (lane == 0 && b) atomicAdd(&cnt[l], __popc(b));
  }
  __syncthreads();
  if (threadIdx.x <= L) counts[(int64_t)blockIdx.x * (L + 1) + threadIdx.x] = cnt[threadIdx.x];
}

// Exclusive prefix, per tree and level, of k_count's per-block box counts
// (in place), one CTA per (tree, level): k_fill reads its block's offsets
// directly (summing the earlier blocks in every k_fill block was quadratic in
// the block count: 170 us of fill at C4's 3.5 M points).
__global__ __launch_bounds__(kBlk) void k_scan_counts(int32_t* __restrict__ counts, int nbx, int nbk, int L) {
  using Scan = cub::BlockScan<int, kBlk>;
  __shared__ typename Scan::TempStorage tmp;
  __shared__ int carry;
  const int tree = blockIdx.x / (L + 1), l = blockIdx.x % (L + 1);
  const int b0 = tree ? nbx : 0, b1 = tree ? nbx + nbk : nbx;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int c = b0; c < b1; c += kBlk) {
    const int b = c + threadIdx.x;
    const int v = b < b1 ? counts[(int64_t)b * (L + 1) + l] : 0;
    int ex, tot;
    Scan(tmp).ExclusiveSum(v, ex, tot);
    if (b < b1) counts[(int64_t)b * (L + 1) + l] = carry + ex;
    __syncthreads();
    if (threadIdx.x == 0) carry += tot;
    __syncthreads();
  }
}

// The plan's box totals and domain flag (nw int64 words) into pinned host
// memory, then seq in word nw (system-scope fences: the host sees the data
// before the flag)
#ifndef SFT_PUBLISH
#define SFT_PUBLISH 1
#endif
__global__ void k_publish(const int64_t* __restrict__ src, int nw, int64_t* dst, int64_t seq) {
  volatile int64_t* d = dst;
  for (int i = threadIdx.x; i < nw; i += blockDim.x) d[i] = src[i];
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    d[nw] = seq;
    __threadfence_system();
  }
}

struct TreeOut {
  uint64_t* key[kMaxLevels];
  int32_t* child_begin[kMaxLevels];
  uint32_t* child_mask[kMaxLevels];
  int32_t* parent[kMaxLevels];
  int32_t* first_pt;
  int32_t* leaf_of;  // [npts] leaf index of each sorted point
  int32_t* perm;
  double* pts_sorted;
  const double* pts;
  int64_t* totals;  // [L+1] box counts per level
};

struct FillArgs {
  TreeOut t[2];
  BlockMap bm;
  int nbk;
};

template <typename KT>
__global__ __launch_bounds__(kBlk) void k_fill(const KT* __restrict__ key, const int32_t* __restrict__ idx,
                                               const uint8_t* __restrict__ ml, const int32_t* __restrict__ counts,
                                               FillArgs A, int d, int L) {
  __shared__ int base[kMaxLevels];
  __shared__ int woff[32][kMaxLevels];
  int tree;
  int64_t ts, lo, hi;
  A.bm.get(blockIdx.x, tree, ts, lo, hi);
  const TreeOut& T = A.t[tree];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int b_last = tree ? A.bm.nbx + A.nbk - 1 : A.bm.nbx - 1;
  // exclusive prefix of the level counts over the earlier blocks of this tree (k_scan_counts)
  if (threadIdx.x <= L) base[threadIdx.x] = counts[(int64_t)blockIdx.x * (L + 1) + threadIdx.x];
  const int64_t i = lo + threadIdx.x;
  const int m = i < hi ? (int)ml[i] : L + 1;
  const unsigned le = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
  for (int l = 0; l <= L; ++l) {
    const unsigned b = __ballot_sync(0xffffffffu, m <= l);
    if (lane == 0) woff[warp][l] = __popc(b);
  }
  __syncthreads();
  if (threadIdx.x <= L) {  // exclusive scan over warps, per level; block total
    int s = 0;
    for (int w = 0; w < 32; ++w) {
      const int v = woff[w][threadIdx.x];
      woff[w][threadIdx.x] = s;
      s += v;
    }
    if ((int)blockIdx.x == b_last) T.totals[threadIdx.x] = base[threadIdx.x] + s;
  }
  __syncthreads();
  const bool valid = i < hi;
  const uint64_t kk = valid ? (uint64_t)key[i] : 0ull;
  const int64_t li = i - ts;  // index within this tree's sorted points
  int bid_prev = -1;
  for (int l = 0; l <= L; ++l) {
    const unsigned b = __ballot_sync(0xffffffffu, m <= l);
    const int bid = base[l] + woff[warp][l] + __popc(b & le) - 1;  // box of point i at level l
    if (m <= l) {  // point i opens box bid at level l (m <= L implies valid)
      const uint64_t kl = (kk >> (d * (L - l))) & ((1ull << (d * l)) - 1ull);
      T.key[l][bid] = kl;
      if (l > 0) {
        T.parent[l][bid] = bid_prev;
        atomicOr(&T.child_mask[l - 1][bid_prev], 1u << (uint32_t)(kl & ((1u << d) - 1u)));
        // the opener of the parent box also opens its first child
        if (m <= l - 1) T.child_begin[l - 1][bid_prev] = bid;
      }
      if (l == L) T.first_pt[bid] = (int32_t)li;
    }
    bid_prev = bid;
  }
  if (!valid) return;
  if (i == hi - 1 && (int)blockIdx.x == b_last) T.first_pt[bid_prev + 1] = (int32_t)(li + 1);
  const int32_t j = idx[i] - (int32_t)ts;
  T.perm[li] = j;
  T.leaf_of[li] = bid_prev;  // box of the point at level L
  for (int a = 0; a < d; ++a) T.pts_sorted[li * d + a] = T.pts[(int64_t)j * d + a];
}

// ------------------------------------------------------------------------
// Small trees (both <= 16K points): the whole build of a tree in one CTA of one
// launch -- child-mask zeroing, Morton keys, the block radix sort, and the
// count / fill steps of k_count / k_fill over the tree's sorted positions in
// chunks of 1024 -- instead of a memset and four launches (small plans are
// latency-bound: every launch boundary costs microseconds).  Same integer
// arithmetic as the multi-kernel path, so identical trees.
// ------------------------------------------------------------------------
struct SmallTreeArgs {
  TreeOut t[2];
  uint32_t* mask[2];     // this tree's child-mask region (zeroed here)
  int64_t mask_words[2];
  void* keys[2];         // [n] sorted keys (scratch: predecessors are read across threads)
  int32_t* idx[2];       // [n] sorted point indices (scratch; !FULL: + the tree's offset, as k_fill reads them)
  int32_t ioff[2];       // that offset (0 when FULL)
  int* err[2];           // domain flag of each tree (1 = a coordinate outside [0,N] or non-finite)
};

// FULL = false: only masks, keys and the sort here (the sorted keys / indices
// written in the layout of the device-wide sort, totals zeroed); k_count and
// k_fill follow with one block per 1024 points.  A single CTA walks its chunks
// one after the other, so the full fusion only pays for small trees.
template <typename KT, int ITEMS, bool FULL>
__global__ __launch_bounds__(1024) void k_small_tree(const double* __restrict__ x, int64_t nx,
                                                     const double* __restrict__ k, int64_t nk, int d, int L, double Nf,
                                                     int64_t N, SmallTreeArgs A) {
  using BRS = cub::BlockRadixSort<KT, 1024, ITEMS, int32_t, SFT_BS_BITS>;
  extern __shared__ __align__(16) unsigned char st_smem[];
  auto& tmp = *reinterpret_cast<typename BRS::TempStorage*>(st_smem);
  __shared__ int cnt[ITEMS][kMaxLevels];  // per 1024-position chunk: boxes opened at each level (then its prefix)
  __shared__ int woff[32][kMaxLevels];
  __shared__ int errf;
  const int tree = blockIdx.x;
  const TreeOut& T = A.t[tree];
  const int64_t n = tree ? nk : nx;
  const double* pts = tree ? k : x;
  KT* const skey = reinterpret_cast<KT*>(A.keys[tree]);
  int32_t* const sidx = A.idx[tree];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
#ifdef SFT_TREE_PROF
  unsigned long long ts[8];
  int nts = 0;
  auto stamp = [&]() { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[nts++])); };
#else
  auto stamp = [&]() {};
#endif
  stamp();
  for (int64_t q = t; q < A.mask_words[tree]; q += 1024) A.mask[tree][q] = 0u;
  if (t == 0) errf = 0;
  for (int q = t; q < ITEMS * kMaxLevels; q += 1024) (&cnt[0][0])[q] = 0;
  __syncthreads();
  // Morton keys of this thread's points (blocked), as k_leaf_keys without the tree bit
  KT kk[ITEMS];
  int32_t vv[ITEMS];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int64_t j = (int64_t)t * ITEMS + i;
    if (j < n) {
      uint64_t c[kMaxDim] = {0, 0, 0};
#pragma unroll
      for (int a = 0; a < kMaxDim; ++a) {
        if (a >= d) break;
        double y = pts[j * d + a];
        if (!(y >= 0.0 && y <= Nf)) {
          bad = true;
          y = 0.0;
        }
        int64_t ci = (int64_t)floor(y);
        if (ci > N - 1) ci = N - 1;
        c[a] = (uint64_t)ci;
      }
      kk[i] = (KT)(d == 2 ? (spread2(c[0]) << 1) | spread2(c[1])
                          : (spread3(c[0]) << 2) | (spread3(c[1]) << 1) | spread3(c[2]));
      vv[i] = (int32_t)j;
    } else {
      kk[i] = ~(KT)0;
      vv[i] = INT32_MAX;
    }
  }
  if (bad) errf = 1;
  stamp();
  BRS(tmp).SortBlockedToStriped(kk, vv, 0, d * L);  // item i of thread t: sorted position i * 1024 + t
#pragma unroll
  for (int i = 0; i < ITEMS; ++i)
    if ((int64_t)i * 1024 + t < n) {
      skey[(int64_t)i * 1024 + t] = kk[i];
      sidx[(int64_t)i * 1024 + t] = vv[i] + A.ioff[tree];
    }
  if constexpr (!FULL) {
    if (t <= L) T.totals[t] = 0;  // (k_fill's last block of the tree writes them)
    __syncthreads();
    if (t == 0) *A.err[tree] = errf;
    return;
  }
  __syncthreads();
  const int nch = (int)((n + 1023) / 1024);  // chunks holding points
  stamp();
  // count: per chunk and level, the boxes its positions open
#pragma unroll 1
  for (int c = 0; c < nch; ++c) {
    const int64_t pos = (int64_t)c * 1024 + t;
    const int m = pos < n ? open_level(skey, pos, 0, d, L) : L + 1;
    for (int l = 0; l <= L; ++l) {
      const unsigned b = __ballot_sync(0xffffffffu, m <= l);
      if (lane == 0 && b) atomicAdd(&cnt[c][l], __popc(b));
    }
  }
  __syncthreads();
  stamp();
  if (t <= L) {  // exclusive prefix over the chunks; the tree's box totals
    int sacc = 0;
    for (int c = 0; c < ITEMS; ++c) {
      const int v = cnt[c][t];
      cnt[c][t] = sacc;
      sacc += v;
    }
    T.totals[t] = sacc;
  }
  __syncthreads();
  // fill, chunk by chunk (k_fill with the chunk prefix as the block base)
  const unsigned le = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
#pragma unroll 1
  for (int c = 0; c < nch; ++c) {
    const int64_t pos = (int64_t)c * 1024 + t;
    const bool valid = pos < n;
    const int m = valid ? open_level(skey, pos, 0, d, L) : L + 1;
    for (int l = 0; l <= L; ++l) {
      const unsigned b = __ballot_sync(0xffffffffu, m <= l);
      if (lane == 0) woff[warp][l] = __popc(b);
    }
    __syncthreads();
    if (t <= L) {
      int sacc = 0;
      for (int w = 0; w < 32; ++w) {
        const int v = woff[w][t];
        woff[w][t] = sacc;
        sacc += v;
      }
    }
    __syncthreads();
    const uint64_t key = valid ? (uint64_t)skey[pos] : 0ull;
    int bid_prev = -1;
    for (int l = 0; l <= L; ++l) {
      const unsigned b = __ballot_sync(0xffffffffu, m <= l);
      const int bid = cnt[c][l] + woff[warp][l] + __popc(b & le) - 1;
      if (m <= l) {
        const uint64_t kl = (key >> (d * (L - l))) & ((1ull << (d * l)) - 1ull);
        T.key[l][bid] = kl;
        if (l > 0) {
          T.parent[l][bid] = bid_prev;
          atomicOr(&T.child_mask[l - 1][bid_prev], 1u << (uint32_t)(kl & ((1u << d) - 1u)));
          if (m <= l - 1) T.child_begin[l - 1][bid_prev] = bid;
        }
        if (l == L) T.first_pt[bid] = (int32_t)pos;
      }
      bid_prev = bid;
    }
    if (valid) {
      if (pos == n - 1) T.first_pt[bid_prev + 1] = (int32_t)n;
      const int32_t j = sidx[pos];
      T.perm[pos] = j;
      T.leaf_of[pos] = bid_prev;
      for (int a = 0; a < d; ++a) T.pts_sorted[pos * d + a] = pts[(int64_t)j * d + a];
    }
    __syncthreads();  // woff is rewritten by the next chunk
  }
  if (t == 0) *A.err[tree] = errf;
  stamp();
#ifdef SFT_TREE_PROF
  if (t == 0)
    printf("[small_tree] tree %d n %lld: zero+keys %.2f sort %.2f count %.2f fill %.2f us\n", tree, (long long)n,
           (ts[1] - ts[0]) * 1e-3, (ts[2] - ts[1]) * 1e-3, (ts[3] - ts[2]) * 1e-3, (ts[4] - ts[3]) * 1e-3);
#endif
}

// ------------------------------------------------------------------------
// Trees of 2K..16K points: one thread-block cluster of CL = 8 CTAs builds a
// tree in one launch.  The sort is a least-significant-digit
// radix sort with 8-bit digits whose keys never leave the cluster's shared
// memory.  CTA r owns the r-th contiguous chunk of the current order.  Per
// digit pass: CTA r ranks its keys by digit, stably (cub::BlockRadixRankMatch,
// keys in warp-striped order = chunk order), publishes its 256 digit counts;
// after a cluster barrier every CTA reads all CTAs' counts over distributed
// shared memory, so a key's place in the whole tree is
//   (keys of smaller digits in the tree) + (keys of its digit in earlier CTAs)
//   + (its rank among its digit in this CTA),
// and it is stored straight into the owner CTA's buffer (DSMEM store); a
// second barrier ends the pass.  Stable like the device-wide sort, so the
// order (and the tree) is identical.  The count and fill steps follow in the
// cluster on the shared-memory-resident sorted chunk (k_count / k_fill with the
// chunk's exclusive prefix over the earlier CTAs, read over DSMEM).  (Measured:
// C1's sort 3 passes ~13 us, count ~4, fill ~7 against ~33 + 4 + 8 for the
// single-CTA sort and the two launches; the same sort with 16-CTA clusters for
// C2 / C3-sized trees (up to 12 items per thread, 4 passes) was slower than
// CUB's onesweep, so those keep the device-wide sort.)
// ------------------------------------------------------------------------
constexpr int kTreeCl = 8;  // CTAs per tree (portable cluster size)
constexpr int kRankBits = 8;
using ClusterRank = cub::BlockRadixRankMatch<1024, kRankBits, false>;

template <typename KT>
struct DigitOf {
  uint32_t shift;
  __device__ __forceinline__ uint32_t Digit(KT k) const { return (uint32_t)(k >> shift) & ((1u << kRankBits) - 1u); }
};

__device__ __forceinline__ int open_level_kv(uint64_t key, uint64_t prev, bool first, int d, int L) {
  if (first) return 0;
  const uint64_t x = key ^ prev;
  if (x == 0) return L + 1;
  return L - (63 - __clzll((long long)x)) / d;
}

template <typename KT, int ITEMS>
constexpr size_t cluster_tree_smem() {
  return (sizeof(typename ClusterRank::TempStorage) + 15) / 16 * 16 + (sizeof(KT) + 4) * ITEMS * 1024;
}

template <typename KT, int ITEMS, int CL>
__global__ __launch_bounds__(1024) void k_cluster_tree(const double* __restrict__ x, int64_t nx,
                                                       const double* __restrict__ k, int64_t nk, int d, int L,
                                                       double Nf, int64_t N, SmallTreeArgs A) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  constexpr int kTile = ITEMS * 1024;
  extern __shared__ __align__(16) unsigned char ct_smem[];
  auto& rtmp = *reinterpret_cast<typename ClusterRank::TempStorage*>(ct_smem);
  KT* const bkey = reinterpret_cast<KT*>(ct_smem + (sizeof(typename ClusterRank::TempStorage) + 15) / 16 * 16);
  int32_t* const bidx = reinterpret_cast<int32_t*>(bkey + kTile);  // (sizeof(KT) * kTile is a multiple of 16)
  __shared__ int s_excl[1 << kRankBits], cnt_s[1 << kRankBits], goff[1 << kRankBits], wsum[8];
  __shared__ int errf;
  const int r = (int)cl.block_rank();
  const int tree = blockIdx.x / CL;
  const TreeOut& T = A.t[tree];
  const int64_t n = tree ? nk : nx;
  const double* pts = tree ? k : x;
  const int64_t chunk = (n + CL - 1) / CL;
  const int64_t lo = min((int64_t)r * chunk, n);
  const int len = (int)(min(lo + chunk, n) - lo);
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
#ifdef SFT_TREE_PROF
  unsigned long long ts[8];
  int nts = 0;
  auto stamp = [&]() { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts[nts++])); };
#else
  auto stamp = [&]() {};
#endif
  stamp();
  for (int64_t q = (int64_t)r * 1024 + t; q < A.mask_words[tree]; q += CL * 1024) A.mask[tree][q] = 0u;
  if (t == 0) errf = 0;
  cl.sync();  // rank 0's errf initialised before any CTA posts to it
  // this CTA's chunk, warp-striped (tile position warp * 32 * ITEMS + i * 32 + lane), Morton keys
  KT kk[ITEMS];
  int32_t vv[ITEMS];
  bool bad = false;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const int tp = warp * 32 * ITEMS + i * 32 + lane;
    if (tp < len) {
      const int64_t g = lo + tp;
      uint64_t c[kMaxDim] = {0, 0, 0};
#pragma unroll
      for (int a = 0; a < kMaxDim; ++a) {
        if (a >= d) break;
        double y = pts[g * d + a];
        if (!(y >= 0.0 && y <= Nf)) {
          bad = true;
          y = 0.0;
        }
        int64_t ci = (int64_t)floor(y);
        if (ci > N - 1) ci = N - 1;
        c[a] = (uint64_t)ci;
      }
      kk[i] = (KT)(d == 2 ? (spread2(c[0]) << 1) | spread2(c[1])
                          : (spread3(c[0]) << 2) | (spread3(c[1]) << 1) | spread3(c[2]));
      vv[i] = (int32_t)g;
    } else {
      kk[i] = ~(KT)0;  // padding: digit 255 in every pass, ranked behind every real key of this CTA
      vv[i] = -1;
    }
  }
  if (bad) atomicOr(cl.map_shared_rank(&errf, 0), 1);
  stamp();
  const int bits = d * L;
  for (int shift = 0; shift < max(bits, 1); shift += kRankBits) {
    int rank[ITEMS];
    int excl[1];
    const DigitOf<KT> dig{(uint32_t)shift};
    ClusterRank(rtmp).RankKeys(kk, rank, dig, excl);
    if (t < (1 << kRankBits)) s_excl[t] = excl[0];
    __syncthreads();
    if (t < (1 << kRankBits))
      cnt_s[t] = (t + 1 < (1 << kRankBits) ? s_excl[t + 1] : kTile) - s_excl[t] -
                 (t + 1 == (1 << kRankBits) ? kTile - len : 0);
    cl.sync();  // every CTA's digit counts published; every CTA has its keys in registers
    int tot = 0, before = 0;
    if (t < (1 << kRankBits)) {
#pragma unroll
      for (int q = 0; q < CL; ++q) {
        const int c = *cl.map_shared_rank(&cnt_s[t], q);
        tot += c;
        before += q < r ? c : 0;
      }
    }
    // exclusive scan of the tree's digit totals over the 256 digits (warps 0..7)
    int inc = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += v;
    }
    if (lane == 31 && warp < 8) wsum[warp] = inc;
    __syncthreads();
    if (t < (1 << kRankBits)) {
      int wpre = 0;
      for (int w = 0; w < warp; ++w) wpre += wsum[w];
      goff[t] = wpre + inc - tot + before - s_excl[t];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (vv[i] >= 0) {
        const int64_t g = goff[dig.Digit(kk[i])] + rank[i];
        const int q = (int)(g / chunk);
        const int o = (int)(g - (int64_t)q * chunk);
        *cl.map_shared_rank(bkey + o, q) = kk[i];
        *cl.map_shared_rank(bidx + o, q) = vv[i];
      }
    }
    cl.sync();  // the pass's keys are in their owners' buffers; no count is read any more
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      const int tp = warp * 32 * ITEMS + i * 32 + lane;
      kk[i] = tp < len ? bkey[tp] : ~(KT)0;
      vv[i] = tp < len ? bidx[tp] : -1;
    }
  }
  stamp();
  if (r == 0 && t == 0) *A.err[tree] = errf;  // (every flag was posted before the first pass barrier)
  {
    // count / fill on the sorted chunk [lo, lo + len) held in bkey / bidx
    __shared__ int cnt[ITEMS][kMaxLevels];
    __shared__ int ctot[kMaxLevels], base[kMaxLevels];
    __shared__ int woff[32][kMaxLevels];
    for (int q = t; q < ITEMS * kMaxLevels; q += 1024) (&cnt[0][0])[q] = 0;
    // the key before this chunk (last of the previous CTA's chunk, full since lo > 0)
    const uint64_t kprev0 = r > 0 && len > 0 ? (uint64_t)*cl.map_shared_rank(bkey + (chunk - 1), r - 1) : 0ull;
    __syncthreads();
    auto ml_at = [&](int j) -> int {
      if (j >= len) return L + 1;
      const uint64_t key = bkey[j];
      const uint64_t prev = j > 0 ? (uint64_t)bkey[j - 1] : kprev0;
      return open_level_kv(key, prev, lo + j == 0, d, L);
    };
    const int nch = (len + 1023) / 1024;
    for (int c = 0; c < nch; ++c) {
      const int m = ml_at(c * 1024 + t);
      for (int l = 0; l <= L; ++l) {
        const unsigned b = __ballot_sync(0xffffffffu, m <= l);
        if (lane == 0 && b) atomicAdd(&cnt[c][l], __popc(b));
      }
    }
    __syncthreads();
    if (t <= L) {
      int sacc = 0;
      for (int c = 0; c < ITEMS; ++c) {
        const int v = cnt[c][t];
        cnt[c][t] = sacc;
        sacc += v;
      }
      ctot[t] = sacc;
    }
    cl.sync();
    if (t <= L) {
      int b = 0;
      for (int q = 0; q < r; ++q) b += *cl.map_shared_rank(&ctot[t], q);
      base[t] = b;
      if (r == CL - 1) T.totals[t] = b + ctot[t];
    }
    cl.sync();  // (no CTA exits while another still reads its ctot / last key)
    stamp();
    const unsigned le = (lane == 31) ? 0xffffffffu : ((2u << lane) - 1u);
    for (int c = 0; c < nch; ++c) {
      const int j = c * 1024 + t;
      const int64_t pos = lo + j;
      const bool valid = j < len;
      const int m = ml_at(j);
      for (int l = 0; l <= L; ++l) {
        const unsigned b = __ballot_sync(0xffffffffu, m <= l);
        if (lane == 0) woff[warp][l] = __popc(b);
      }
      __syncthreads();
      if (t <= L) {
        int sacc = 0;
        for (int w = 0; w < 32; ++w) {
          const int v = woff[w][t];
          woff[w][t] = sacc;
          sacc += v;
        }
      }
      __syncthreads();
      const uint64_t key = valid ? (uint64_t)bkey[j] : 0ull;
      int bid_prev = -1;
      for (int l = 0; l <= L; ++l) {
        const unsigned b = __ballot_sync(0xffffffffu, m <= l);
        const int bid = base[l] + cnt[c][l] + woff[warp][l] + __popc(b & le) - 1;
        if (m <= l) {
          const uint64_t kl = (key >> (d * (L - l))) & ((1ull << (d * l)) - 1ull);
          T.key[l][bid] = kl;
          if (l > 0) {
            T.parent[l][bid] = bid_prev;
            atomicOr(&T.child_mask[l - 1][bid_prev], 1u << (uint32_t)(kl & ((1u << d) - 1u)));
            if (m <= l - 1) T.child_begin[l - 1][bid_prev] = bid;
          }
          if (l == L) T.first_pt[bid] = (int32_t)pos;
        }
        bid_prev = bid;
      }
      if (valid) {
        if (pos == n - 1) T.first_pt[bid_prev + 1] = (int32_t)n;
        const int32_t jj = bidx[j];
        T.perm[pos] = jj;
        T.leaf_of[pos] = bid_prev;
        for (int a = 0; a < d; ++a) T.pts_sorted[pos * d + a] = pts[(int64_t)jj * d + a];
      }
      __syncthreads();  // woff is rewritten by the next chunk
    }
    stamp();
#ifdef SFT_TREE_PROF
    if (t == 0 && (r == 0 || r == CL - 1))
      printf("[cluster_tree] tree %d rank %d n %lld: zero+keys %.2f sort %.2f count %.2f fill %.2f us\n", tree, r,
             (long long)n, (ts[1] - ts[0]) * 1e-3, (ts[2] - ts[1]) * 1e-3, (ts[3] - ts[2]) * 1e-3,
             (ts[4] - ts[3]) * 1e-3);
#endif
  }
}

static inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// CUB radix-sort tuning for the tree build: the onesweep digit width (the
// keys have d*L (+1) <= 29 bits at the BASELINE configs, so 10-bit digits need
// 3 passes where CUB's default 8-bit digits need 4) and items per thread.
// Everything else as CUB's SM100 policy.
#ifndef SFT_SORT_BITS
#define SFT_SORT_BITS 8
#endif
#ifndef SFT_SORT_ITEMS
#define SFT_SORT_ITEMS 12  // C2 plan -8 us vs CUB's 23 (more, shorter tiles for ~150K keys)
#endif
#ifndef SFT_SORT_THREADS
#define SFT_SORT_THREADS 384
#endif
template <typename KeyT, typename ValueT, typename OffsetT>
struct SortHub {
  using DominantT = ::cuda::std::_If<(sizeof(ValueT) > sizeof(KeyT)), ValueT, KeyT>;
  struct Policy1000 : cub::ChainedPolicy<1000, Policy1000, Policy1000> {
    static constexpr bool ONESWEEP = true;
    static constexpr int ONESWEEP_RADIX_BITS = SFT_SORT_BITS;
    using HistogramPolicy = cub::AgentRadixSortHistogramPolicy<128, 16, 1, KeyT, ONESWEEP_RADIX_BITS>;
    using ExclusiveSumPolicy = cub::AgentRadixSortExclusiveSumPolicy<256, ONESWEEP_RADIX_BITS>;
    using OnesweepPolicy =
        cub::AgentRadixSortOnesweepPolicy<SFT_SORT_THREADS, SFT_SORT_ITEMS, DominantT, 1, cub::RADIX_RANK_MATCH_EARLY_COUNTS_ANY,
                                          cub::BLOCK_SCAN_RAKING_MEMOIZE, cub::RADIX_SORT_STORE_DIRECT,
                                          ONESWEEP_RADIX_BITS>;
    using ScanPolicy = cub::AgentScanPolicy<512, 23, OffsetT, cub::BLOCK_LOAD_WARP_TRANSPOSE, cub::LOAD_DEFAULT,
                                            cub::BLOCK_STORE_WARP_TRANSPOSE, cub::BLOCK_SCAN_RAKING_MEMOIZE>;
    using DownsweepPolicy =
        cub::AgentRadixSortDownsweepPolicy<512, 23, DominantT, cub::BLOCK_LOAD_TRANSPOSE, cub::LOAD_DEFAULT,
                                           cub::RADIX_RANK_MATCH, cub::BLOCK_SCAN_WARP_SCANS, 7>;
    using AltDownsweepPolicy =
        cub::AgentRadixSortDownsweepPolicy<256, 47, DominantT, cub::BLOCK_LOAD_TRANSPOSE, cub::LOAD_DEFAULT,
                                           cub::RADIX_RANK_MEMOIZE, cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using UpsweepPolicy = cub::AgentRadixSortUpsweepPolicy<256, 23, DominantT, cub::LOAD_DEFAULT, 7>;
    using AltUpsweepPolicy = cub::AgentRadixSortUpsweepPolicy<256, 47, DominantT, cub::LOAD_DEFAULT, 6>;
    using SingleTilePolicy =
        cub::AgentRadixSortDownsweepPolicy<256, 19, DominantT, cub::BLOCK_LOAD_DIRECT, cub::LOAD_LDG,
                                           cub::RADIX_RANK_MEMOIZE, cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using SegmentedPolicy =
        cub::AgentRadixSortDownsweepPolicy<192, 39, DominantT, cub::BLOCK_LOAD_TRANSPOSE, cub::LOAD_DEFAULT,
                                           cub::RADIX_RANK_MEMOIZE, cub::BLOCK_SCAN_WARP_SCANS, 6>;
    using AltSegmentedPolicy =
        cub::AgentRadixSortDownsweepPolicy<384, 11, DominantT, cub::BLOCK_LOAD_TRANSPOSE, cub::LOAD_DEFAULT,
                                           cub::RADIX_RANK_MEMOIZE, cub::BLOCK_SCAN_WARP_SCANS, 5>;
  };
  using MaxPolicy = Policy1000;
};
template <typename KT>
static cudaError_t sort_pairs(void* temp, size_t& bytes, const KT* kin, KT* kout, const int32_t* iin, int32_t* iout,
                              int n, int bits, cudaStream_t s) {
  cub::DoubleBuffer<KT> dk(const_cast<KT*>(kin), kout);
  cub::DoubleBuffer<int32_t> dv(const_cast<int32_t*>(iin), iout);
  return cub::DispatchRadixSort<false, KT, int32_t, int, SortHub<KT, int32_t, int>>::Dispatch(
      temp, bytes, dk, dv, n, 0, bits, false, s);
}

// Per-thread cache of the tree-build scratch and of an instantiated CUDA graph
// of the CUB radix sort for one (point count, key bits, key type): plans built
// back to back with the same sizes replay the graph (a few us of host time
// instead of ~50 us of CUB dispatch, during which the GPU idles).  The scratch
// is only used before sft_plan's counts sync, so consecutive plans of one
// thread never overlap on it.  SFT_SORT_GRAPH=0 disables (plain CUB call).
struct SortCache {
  int64_t n = -1, nx = -1;  // the graph sorts [0, nx) and [nx, n) as two branches: nx is part of the key
  int bits = -1, ksz = 0, nb = -1, L = -1, dev = -1;
  char* scr = nullptr;
  cudaGraphExec_t exec = nullptr;
};
static thread_local SortCache g_sort;
static bool sort_graph_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SFT_SORT_GRAPH");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

#define CK(x)                                                            \
  do {                                                                   \
    cudaError_t e_ = (x);                                                \
    if (e_ != cudaSuccess) {                                             \
      if (err) *err = std::string(#x) + ": " + cudaGetErrorString(e_);   \
      return SFT_E_CUDA;                                                 \
    }                                                                    \
  } while (0)

static size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// upper bound on the non-empty boxes of a tree with n points at level l
static int64_t level_cap(int64_t n, int d, int l) {
  if (d * l >= 40) return n;
  return std::min<int64_t>(n, int64_t(1) << (d * l));
}

static bool small_tree_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SFT_SMALL_TREE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
// both trees built by k_small_tree (one launch, no memset of the child masks)
template <typename KT>
static bool small_tree_path(int64_t nx, int64_t nk) {
  constexpr bool bs_fits =
      sizeof(typename cub::BlockRadixSort<KT, 1024, kBlockSortItems, int32_t, SFT_BS_BITS>::TempStorage) <= 200 * 1024;
  return bs_fits && nx <= kBlockSortMax && nk <= kBlockSortMax && sort_graph_enabled() && small_tree_enabled();
}

static bool cluster_tree_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SFT_CLUSTER_TREE");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}
// full fusion (count / fill inside the sort CTA) up to this many points per tree
static int64_t small_full_max() {
  static int64_t v = -1;
  if (v < 0) {
    const char* e = getenv("SFT_SMALL_FULL");
    v = e ? atoll(e) : 2048;
  }
  return v;
}

template <typename KT, bool FULL>
static cudaError_t launch_small_tree(const SmallTreeArgs& A, const double* x_dev, int64_t nx, const double* k_dev,
                                     int64_t nk, int d, int L, int64_t N, cudaStream_t s) {
  const int64_t nmax = std::max(nx, nk);
  auto run = [&](auto items) -> cudaError_t {
    constexpr int IT = decltype(items)::value;
    using BRS = cub::BlockRadixSort<KT, 1024, IT, int32_t, SFT_BS_BITS>;
    const size_t bsm = sizeof(typename BRS::TempStorage);
    static PerDevice<int> attr;  // the shared-memory opt-in, once per device and instantiation
    int one = 0;
    cudaError_t e = attr.get(&one, [&](int, int* v) {
      *v = 1;
      return cudaFuncSetAttribute(k_small_tree<KT, IT, FULL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
    });
    if (e != cudaSuccess) return e;
    k_small_tree<KT, IT, FULL><<<2, 1024, bsm, s>>>(x_dev, nx, k_dev, nk, d, L, (double)N, N, A);
    return cudaGetLastError();
  };
  cudaError_t e;
  if (nmax <= 1024) e = run(std::integral_constant<int, 1>());
  else if (nmax <= 2048) e = run(std::integral_constant<int, 2>());
  else if (nmax <= 4096) e = run(std::integral_constant<int, 4>());
  else if (nmax <= 8192) e = run(std::integral_constant<int, 8>());
  else if (nmax <= 11264) e = run(std::integral_constant<int, 11>());
  else e = run(std::integral_constant<int, kBlockSortItems>());
  count_launch();
  return e;
}

// cluster tree build (k_cluster_tree, 8 CTAs per tree): items per thread for
// trees of nmax points, or 0 when the path does not apply (more than 16K
// points, disabled, or the cluster cannot be scheduled on this device)
template <typename KT, int IT>
static cudaError_t cluster_config(cudaLaunchConfig_t* cfg, cudaLaunchAttribute* at, cudaStream_t s) {
  const size_t bsm = cluster_tree_smem<KT, IT>();
  static PerDevice<int> attr;  // the shared-memory opt-in, once per device and instantiation
  int one = 0;
  cudaError_t e = attr.get(&one, [&](int, int* v) {
    *v = 1;
    return cudaFuncSetAttribute(k_cluster_tree<KT, IT, kTreeCl>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)bsm);
  });
  if (e != cudaSuccess) return e;
  *cfg = cudaLaunchConfig_t{};
  cfg->gridDim = dim3(2 * kTreeCl);
  cfg->blockDim = dim3(1024);
  cfg->dynamicSmemBytes = bsm;
  cfg->stream = s;
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kTreeCl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg->attrs = at;
  cfg->numAttrs = 1;
  return cudaSuccess;
}
template <typename KT, typename F>
static cudaError_t cluster_dispatch(int items, F&& f) {
  if (items == 1) return f(std::integral_constant<int, 1>());
  if (items == 2) return f(std::integral_constant<int, 2>());
  return cudaErrorInvalidConfiguration;
}
template <typename KT>
static int cluster_tree_items(int64_t nx, int64_t nk) {
  if (!cluster_tree_enabled() || !sort_graph_enabled() || !small_tree_enabled()) return 0;
  const int64_t nmax = std::max(nx, nk);
  const int items = nmax <= kTreeCl * 1024 ? 1 : nmax <= kTreeCl * 2048 ? 2 : 0;
  if (!items) return 0;
  static PerDevice<int> ok[2];  // clusters of this instantiation schedulable on the device
  int v = 0;
  cudaError_t e = ok[items - 1].get(&v, [&](int, int* r) {
    *r = 0;
    cluster_dispatch<KT>(items, [&](auto it) -> cudaError_t {
      constexpr int IT = decltype(it)::value;
      cudaLaunchConfig_t cfg;
      cudaLaunchAttribute at[1];
      cudaError_t e3 = cluster_config<KT, IT>(&cfg, at, 0);
      int nc = 0;
      if (e3 == cudaSuccess) e3 = cudaOccupancyMaxActiveClusters(&nc, k_cluster_tree<KT, IT, kTreeCl>, &cfg);
      *r = (e3 == cudaSuccess && nc >= 1) ? 1 : 0;
      return cudaSuccess;
    });
    cudaGetLastError();  // a refused configuration only disables the path
    return cudaSuccess;
  });
  return (e == cudaSuccess && v) ? items : 0;
}
template <typename KT>
static cudaError_t launch_cluster_tree(int items, const SmallTreeArgs& A, const double* x_dev, int64_t nx,
                                       const double* k_dev, int64_t nk, int d, int L, int64_t N, cudaStream_t s) {
  cudaError_t e = cluster_dispatch<KT>(items, [&](auto it) -> cudaError_t {
    constexpr int IT = decltype(it)::value;
    cudaLaunchConfig_t cfg;
    cudaLaunchAttribute at[1];
    cudaError_t e1 = cluster_config<KT, IT>(&cfg, at, s);
    if (e1 != cudaSuccess) return e1;
    return cudaLaunchKernelEx(&cfg, k_cluster_tree<KT, IT, kTreeCl>, x_dev, nx, k_dev, nk, d, L, (double)N, N, A);
  });
  count_launch();
  return e;
}

template <typename KT>
static int sort_and_fill(sft_plan_s* P, const double* x_dev, const double* k_dev, char* arena,
                         const std::vector<size_t>* o_key, const std::vector<size_t>* o_par,
                         const std::vector<size_t>* o_cm, const std::vector<size_t>* o_cb, const size_t* o_first,
                         const size_t* o_leafof, const size_t* o_perm, const size_t* o_pts, const size_t* o_tot,
                         const double* const* src, char** scr_out, size_t* scr_bytes, FillArgs& fa,
                         std::string* err) {
  cudaStream_t s = P->stream;
  const int d = P->d, L = P->L;
  const int64_t nx = P->nx, nk = P->nk, n = nx + nk;
  // ---- scratch ----
  const int nbx = (int)nblk(nx, kBlk), nbk = (int)nblk(nk, kBlk);
  const int bits = d * L + 1;
  SortCache& C = g_sort;
  // trees of <= kBlockSortMax points: one block-sort launch; larger: the cached
  // graph of the device-wide sort (or the plain call, SFT_SORT_GRAPH=0)
  constexpr bool bs_fits =
      sizeof(typename cub::BlockRadixSort<KT, 1024, kBlockSortItems, int32_t, SFT_BS_BITS>::TempStorage) <= 200 * 1024;
  const int64_t nmax = std::max(nx, nk);
  const bool small = small_tree_path<KT>(nx, nk);
  // 2K..16K points: the whole build in one cluster launch (k_cluster_tree)
  const int citems = (small && nmax <= small_full_max()) ? 0 : cluster_tree_items<KT>(nx, nk);
  const bool block_sort = bs_fits && nx <= kBlockSortMax && nk <= kBlockSortMax && sort_graph_enabled();
  const bool use_graph = sort_graph_enabled() && n >= 4096 && !block_sort;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  auto fill_out = [&](TreeOut& o, int t) {
    for (int l = 0; l < kMaxLevels; ++l) {
      const bool ok = l <= L;
      o.key[l] = ok ? (uint64_t*)(arena + o_key[t][l]) : nullptr;
      o.parent[l] = ok ? (int32_t*)(arena + o_par[t][l]) : nullptr;
      o.child_mask[l] = ok ? (uint32_t*)(arena + o_cm[t][l]) : nullptr;
      o.child_begin[l] = ok ? (int32_t*)(arena + o_cb[t][l]) : nullptr;
    }
    o.first_pt = (int32_t*)(arena + o_first[t]);
    o.leaf_of = (int32_t*)(arena + o_leafof[t]);
    o.perm = (int32_t*)(arena + o_perm[t]);
    o.pts_sorted = (double*)(arena + o_pts[t]);
    o.pts = src[t];
    o.totals = (int64_t*)(arena + o_tot[t]);
  };
  auto small_args = [&](SmallTreeArgs& A) {
    for (int t = 0; t < 2; ++t) {
      fill_out(A.t[t], t);
      A.mask[t] = (uint32_t*)(arena + o_cm[t][0]);
      A.mask_words[t] = (int64_t)(o_cm[t][L] + 4 * level_cap(t ? nk : nx, d, L) - o_cm[t][0]) / 4;
      A.err[t] = P->d_err + t;  // the two halves of the header's error word
    }
  };
  if (citems) {
    const size_t so = align_up(sizeof(KT) * n, 256) + 4 * n;
    char* scr = nullptr;
    CK(block_alloc((void**)&scr, so, s));
    SmallTreeArgs A;
    small_args(A);
    for (int t = 0; t < 2; ++t) fa.t[t] = A.t[t];
    A.keys[0] = scr;
    A.keys[1] = scr + sizeof(KT) * nx;
    A.idx[0] = (int32_t*)(scr + align_up(sizeof(KT) * n, 256));
    A.idx[1] = A.idx[0] + nx;
    A.ioff[0] = A.ioff[1] = 0;
    CK(launch_cluster_tree<KT>(citems, A, x_dev, nx, k_dev, nk, d, L, P->N, s));
    trace_mark("cluster_tree", s, true);
    *scr_out = scr;
    *scr_bytes = so;
    return SFT_OK;
  }
  if (small && nmax <= small_full_max()) {
    if constexpr (bs_fits) {
      const size_t so = align_up(sizeof(KT) * n, 256) + 4 * n;
      char* scr = nullptr;
      CK(block_alloc((void**)&scr, so, s));
      SmallTreeArgs A;
      small_args(A);
      for (int t = 0; t < 2; ++t) fa.t[t] = A.t[t];
      A.keys[0] = scr;
      A.keys[1] = scr + sizeof(KT) * nx;
      A.idx[0] = (int32_t*)(scr + align_up(sizeof(KT) * n, 256));
      A.idx[1] = A.idx[0] + nx;
      A.ioff[0] = A.ioff[1] = 0;
      CK((launch_small_tree<KT, true>(A, x_dev, nx, k_dev, nk, d, L, P->N, s)));
      trace_mark("small_tree", s, true);
      *scr_out = scr;
      *scr_bytes = so;
      return SFT_OK;
    }
  }
  const bool hit = use_graph && C.exec && C.n == n && C.nx == nx && C.bits == bits && C.ksz == (int)sizeof(KT) &&
                   C.nb == nbx + nbk && C.L == L && C.dev == dev;
  // graph path: X and K sorted as two parallel branches (disjoint halves of the
  // key array, the tree bit is constant in each; each sort is latency-bound, so
  // two half-size sorts side by side take ~60% of one full-size sort)
  size_t cub_bytes = 0, cub_x = 0, cub_k = 0;
  if (!hit && !use_graph && !block_sort)
    CK(cub::DeviceRadixSort::SortPairs(nullptr, cub_bytes, (KT*)nullptr, (KT*)nullptr, (int32_t*)nullptr,
                                       (int32_t*)nullptr, (int)n, 0, bits, s));
  if (use_graph) {
    CK(sort_pairs<KT>(nullptr, cub_x, (KT*)nullptr, (KT*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr, (int)nx,
                      bits - 1, s));
    CK(sort_pairs<KT>(nullptr, cub_k, (KT*)nullptr, (KT*)nullptr, (int32_t*)nullptr, (int32_t*)nullptr, (int)nk,
                      bits - 1, s));
    cub_bytes = align_up(cub_x, 256) + cub_k;
  }
  size_t so = 0;
  const size_t s_kin = so;
  so = align_up(so + sizeof(KT) * n, 256);
  const size_t s_kout = so;
  so = align_up(so + sizeof(KT) * n, 256);
  const size_t s_iin = so;
  so = align_up(so + 4 * n, 256);
  const size_t s_iout = so;
  so = align_up(so + 4 * n, 256);
  const size_t s_ml = so;
  so = align_up(so + n, 256);
  const size_t s_cnt = so;
  so = align_up(so + 4 * (size_t)(nbx + nbk) * (L + 1), 256);
  const size_t s_cub = so;
  so = align_up(so + cub_bytes, 256);
  char* scr = nullptr;
  if (hit) {
    scr = C.scr;  // same sizes and offsets as when the graph was captured
  } else if (use_graph) {
    // (re)build the cached scratch and capture the sort into a graph
    if (C.exec) cudaGraphExecDestroy(C.exec);
    if (C.scr) cudaFree(C.scr);  // synchronises: nothing of the old scratch is in flight
    C = SortCache();
    CK(cudaMalloc((void**)&C.scr, so));
    scr = C.scr;
  } else {
    CK(block_alloc((void**)&scr, so, s));
  }
  trace_mark("scr", s, true);
  KT* keys_in = (KT*)(scr + s_kin);
  KT* keys_out = (KT*)(scr + s_kout);
  int32_t* idx_in = (int32_t*)(scr + s_iin);
  int32_t* idx_out = (int32_t*)(scr + s_iout);
  uint8_t* ml = (uint8_t*)(scr + s_ml);
  int32_t* counts = (int32_t*)(scr + s_cnt);

  if (small) {  // masks + keys + block sort in one launch; k_count / k_fill below
    if constexpr (bs_fits) {
      SmallTreeArgs A;
      small_args(A);
      A.keys[0] = keys_out;
      A.keys[1] = keys_out + nx;
      A.idx[0] = idx_out;
      A.idx[1] = idx_out + nx;
      A.ioff[0] = 0;
      A.ioff[1] = (int32_t)nx;
      CK((launch_small_tree<KT, false>(A, x_dev, nx, k_dev, nk, d, L, P->N, s)));
    }
  } else {
    k_leaf_keys<KT><<<nblk(n, 256), 256, 0, s>>>(x_dev, nx, k_dev, nk, d, L, (double)P->N, P->N, keys_in, idx_in,
                                                 P->d_err);
    count_launch();
    CK(cudaGetLastError());
  }
  trace_mark("keys", s, true);
  if (small) {
  } else if (block_sort) {
    if constexpr (bs_fits) {
      const int64_t nmax = std::max(nx, nk);
      auto run = [&](auto items) -> cudaError_t {
        constexpr int IT = decltype(items)::value;
        using BRS = cub::BlockRadixSort<KT, 1024, IT, int32_t, SFT_BS_BITS>;
        const size_t bsm = sizeof(typename BRS::TempStorage);
        static PerDevice<int> attr;  // the shared-memory opt-in, once per device and instantiation
        int one = 0;
        cudaError_t e = attr.get(&one, [&](int, int* v) {
          *v = 1;
          return cudaFuncSetAttribute(k_block_sort<KT, IT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bsm);
        });
        if (e != cudaSuccess) return e;
        // (the tree bit above bit d*L is constant within a tree)
        k_block_sort<KT, IT><<<2, 1024, bsm, s>>>(keys_in, idx_in, keys_out, idx_out, nx, nk, bits - 1);
        return cudaGetLastError();
      };
      cudaError_t e;
      if (nmax <= 1024) e = run(std::integral_constant<int, 1>());
      else if (nmax <= 2048) e = run(std::integral_constant<int, 2>());
      else if (nmax <= 4096) e = run(std::integral_constant<int, 4>());
      else if (nmax <= 8192) e = run(std::integral_constant<int, 8>());
      else if (nmax <= 11264) e = run(std::integral_constant<int, 11>());
      else e = run(std::integral_constant<int, kBlockSortItems>());
      count_launch();
      CK(e);
    }
  } else if (!use_graph) {
    CK(cub::DeviceRadixSort::SortPairs(scr + s_cub, cub_bytes, keys_in, keys_out, idx_in, idx_out, (int)n, 0, bits, s));
  } else {
    if (!hit) {
      cudaStream_t cs = nullptr, cs2 = nullptr;
      cudaEvent_t fork = nullptr, join = nullptr;
      CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      CK(cudaStreamCreateWithFlags(&cs2, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
      CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      cudaEventRecord(fork, cs);
      cudaStreamWaitEvent(cs2, fork, 0);
      const size_t ox = align_up(cub_x, 256);
      cudaError_t ce = sort_pairs<KT>(scr + s_cub, cub_x, keys_in, keys_out, idx_in, idx_out, (int)nx, bits - 1, cs);
      cudaError_t ce3 = sort_pairs<KT>(scr + s_cub + ox, cub_k, keys_in + nx, keys_out + nx, idx_in + nx, idx_out + nx,
                                       (int)nk, bits - 1, cs2);
      cudaEventRecord(join, cs2);
      cudaStreamWaitEvent(cs, join, 0);
      cudaGraph_t g = nullptr;
      cudaError_t ce2 = cudaStreamEndCapture(cs, &g);
      cudaStreamDestroy(cs);
      cudaStreamDestroy(cs2);
      cudaEventDestroy(fork);
      cudaEventDestroy(join);
      CK(ce);
      CK(ce3);
      CK(ce2);
      ce = cudaGraphInstantiate(&C.exec, g, 0);
      cudaGraphDestroy(g);
      CK(ce);
      C.n = n;
      C.nx = nx;
      C.bits = bits;
      C.ksz = (int)sizeof(KT);
      C.nb = nbx + nbk;
      C.L = L;
      C.dev = dev;
    }
    CK(cudaGraphLaunch(C.exec, s));
  }
  trace_mark("sort", s, true);
  BlockMap bm{nx, n, nbx};
  k_count<KT><<<nbx + nbk, kBlk, 0, s>>>(keys_out, bm, d, L, ml, counts);
  count_launch();
  CK(cudaGetLastError());
  k_scan_counts<<<2 * (L + 1), kBlk, 0, s>>>(counts, nbx, nbk, L);
  count_launch();
  CK(cudaGetLastError());
  trace_mark("count", s, true);

  fa.bm = bm;
  fa.nbk = nbk;
  for (int t = 0; t < 2; ++t) fill_out(fa.t[t], t);
  k_fill<KT><<<nbx + nbk, kBlk, 0, s>>>(keys_out, idx_out, ml, counts, fa, d, L);
  count_launch();
  CK(cudaGetLastError());
  trace_mark("fill", s, true);

  *scr_out = use_graph ? nullptr : scr;  // the cached scratch is not the plan's to free
  *scr_bytes = so;
  return SFT_OK;
}

int build_trees(sft_plan_s* P, const double* x_dev, const double* k_dev, std::string* err) {
  cudaStream_t s = P->stream;
  const int d = P->d, L = P->L;
  const int64_t nx = P->nx, nk = P->nk;
  if (L + 1 > kMaxLevels) {
    if (err) *err = "tree depth exceeds kMaxLevels";
    return SFT_E_ARG;
  }
  Tree* trees[2] = {&P->X, &P->K};
  const int64_t npt[2] = {nx, nk};
  const double* src[2] = {x_dev, k_dev};

  // ---- persistent arena: level arrays (upper bounds) + sorted points ----
  size_t off = 0;
  std::vector<size_t> o_key[2], o_cb[2], o_cm[2], o_par[2];
  size_t o_first[2], o_leafof[2], o_perm[2], o_pts[2], o_tot[2];
  size_t cm_lo = 0, cm_hi = 0;
  for (int t = 0; t < 2; ++t) {
    o_key[t].resize(L + 1);
    o_par[t].resize(L + 1);
    for (int l = 0; l <= L; ++l) {
      o_key[t][l] = off;
      off = align_up(off + 8 * level_cap(npt[t], d, l), 256);
      o_par[t][l] = off;
      off = align_up(off + 4 * level_cap(npt[t], d, l), 256);
    }
  }
  // per-tree box totals [2][L+1] and the domain-error flag, then the child
  // masks of both trees: one memset zeroes all of it, one copy reads it back
  const size_t o_hdr = off;
  cm_lo = off;
  o_tot[0] = off;
  o_tot[1] = off + 8 * (L + 1);
  const size_t o_errf = off + 16 * (L + 1);
  off = align_up(off + 16 * (L + 1) + 8, 256);
  for (int t = 0; t < 2; ++t) {
    o_cm[t].resize(L + 1);
    for (int l = 0; l <= L; ++l) {
      o_cm[t][l] = off;
      off = align_up(off + 4 * level_cap(npt[t], d, l), 256);
    }
  }
  cm_hi = off;
  for (int t = 0; t < 2; ++t) {
    o_cb[t].resize(L + 1);
    for (int l = 0; l <= L; ++l) {
      o_cb[t][l] = off;
      off = align_up(off + 4 * level_cap(npt[t], d, l), 256);
    }
    o_first[t] = off;
    off = align_up(off + 4 * (level_cap(npt[t], d, L) + 1), 256);
    o_leafof[t] = off;
    off = align_up(off + 4 * npt[t], 256);
    o_perm[t] = off;
    off = align_up(off + 4 * npt[t], 256);
    o_pts[t] = off;
    off = align_up(off + 8 * d * npt[t], 256);
  }
  char* arena = nullptr;
  CK(block_alloc((void**)&arena, off, s));
  trace_mark("alloc", s, true);
  P->X.arena = arena;
  P->X.arena_bytes = off;
  P->K.arena = nullptr;
  // (the small-tree and cluster kernels zero their masks and write the whole header themselves)
  const bool small = (d * L + 1 <= 32) ? small_tree_path<uint32_t>(nx, nk) : small_tree_path<uint64_t>(nx, nk);
  if (!small) CK(cudaMemsetAsync(arena + cm_lo, 0, cm_hi - cm_lo, s));
  P->d_err = (int*)(arena + o_errf);  // lives in the arena (freed with the trees)
  trace_mark("arena", s, true);

  // ---- sort + fill (32-bit point keys when d*L+1 <= 32) ----
  char* scr = nullptr;
  size_t scr_bytes = 0;
  FillArgs fa;
  int rc = (d * L + 1 <= 32)
               ? sort_and_fill<uint32_t>(P, x_dev, k_dev, arena, o_key, o_par, o_cm, o_cb, o_first, o_leafof, o_perm,
                                         o_pts, o_tot, src, &scr, &scr_bytes, fa, err)
               : sort_and_fill<uint64_t>(P, x_dev, k_dev, arena, o_key, o_par, o_cm, o_cb, o_first, o_leafof, o_perm,
                                         o_pts, o_tot, src, &scr, &scr_bytes, fa, err);
  if (rc) return rc;

  trace_mark("enq");
  // ---- the one host sync: exact box counts + domain error flag ----
  // k_publish writes them into pinned host memory (through its UVA address)
  // followed by a sequence flag the host spins on -- the kernel's completion
  // is seen a few us sooner than a D2H copy + stream synchronisation (the
  // host polls the stream now and then: a failed launch cannot hang it)
  static thread_local int64_t* h = nullptr;
  static thread_local int64_t seq = 0;
  if (!h) CK(cudaMallocHost((void**)&h, (2 * kMaxLevels + 2) * sizeof(int64_t)));
  const int nw = 2 * (L + 1) + 1;
#if !SFT_PUBLISH  // (A/B: D2H copy + stream synchronisation)
  CK(cudaMemcpyAsync(h, arena + o_hdr, nw * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
  if (scr) block_free(scr, scr_bytes, s);
  CK(cudaStreamSynchronize(s));
  (void)seq;
#else
  volatile int64_t* hv = h;
  hv[nw] = 0;
  ++seq;
  k_publish<<<1, 64, 0, s>>>(reinterpret_cast<const int64_t*>(arena + o_hdr), nw, h, seq);
  count_launch();
  CK(cudaGetLastError());
  if (scr) block_free(scr, scr_bytes, s);
  for (long it = 1; hv[nw] != seq; ++it) {
    if ((it & 255) == 0) {
      const cudaError_t q = cudaStreamQuery(s);
      if (q != cudaErrorNotReady && hv[nw] != seq) {
        if (err) *err = std::string("tree build: ") + (q == cudaSuccess ? "header not published" : cudaGetErrorString(q));
        return SFT_E_CUDA;
      }
    }
  }
  std::atomic_thread_fence(std::memory_order_acquire);
#endif
  trace_mark("sync");
  const bool herr = h[2 * (L + 1)] != 0;  // either half (the small-tree path flags each tree)
  if (herr) {
    if (err) *err = "a coordinate is non-finite or outside [0,N]";
    return SFT_E_DOMAIN;
  }
  for (int t = 0; t < 2; ++t) {
    Tree& T = *trees[t];
    T.d = d;
    T.L = L;
    T.npts = npt[t];
    T.lev.assign(L + 1, TreeLevel());
    T.counts.assign(L + 1, 0);
    for (int l = 0; l <= L; ++l) {
      TreeLevel& lv = T.lev[l];
      lv.n = T.counts[l] = h[t * (L + 1) + l];
      lv.key = fa.t[t].key[l];
      lv.parent = l > 0 ? fa.t[t].parent[l] : nullptr;
      lv.child_mask = l < L ? fa.t[t].child_mask[l] : nullptr;
      lv.child_begin = l < L ? fa.t[t].child_begin[l] : nullptr;
    }
    T.first_pt = fa.t[t].first_pt;
    T.leaf_of = fa.t[t].leaf_of;
    T.perm = fa.t[t].perm;
    T.pts_sorted = fa.t[t].pts_sorted;
  }
  return SFT_OK;
}

void free_tree(Tree& T, cudaStream_t s) {
  if (T.arena) block_free(T.arena, T.arena_bytes, s);
  T.arena = nullptr;
  T.lev.clear();
  T.first_pt = nullptr;
  T.perm = nullptr;
  T.pts_sorted = nullptr;
}

}  // namespace sft
