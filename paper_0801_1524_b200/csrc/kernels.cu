// kernels.cu -- steps 2-4 of the butterfly as sm_100a FP64
// kernels in the box-relative h-representation (sft_internal.cuh).
//
//   K2 leaf:        h^{A0 B}_m = sum_{k_j in B} f_j e^{i pi sum s} prod_ax r_{m_ax}(s_ax)
//   K3 translation: h^{AB} = sum_{present B_c} (x)_ax T[alpha_ax][beta_ax] h^{A' B_c}
//                   T[a][b] = c_ab (RC_b + i (2a-1) RS_b) with RC/RS real p x p in the
//                   constant bank (immediate DFMA operands); one CTA = G groups
//                   (A', B); the <= 2^d child arrays of each group are staged
//                   into shared memory with 1-D TMA bulk copies (cp.async.bulk +
//                   mbarrier); the sum over children is factorised axis by axis,
//                   in place in shared memory; the last axis pass stores the
//                   <= 2^d parent arrays straight to HBM (coalesced).
//   K4 final:       u_i = sum_l prod_ax e^{i pi l_ax (2 xi_ax - 1)/(p-1)} h^{A B0}_l
//
// No floating-point atomics: every output is produced by one thread in a fixed
// order, so results are bitwise reproducible.
#include <algorithm>
#include <atomic>

#include "sft_internal.cuh"

namespace sft {

static std::atomic<long long> g_launches{0};
void count_launch(int n) { g_launches += n; }
long long launch_count() { return g_launches.load(); }

template <int B, int E>
struct Pow {
  static constexpr int v = B * Pow<B, E - 1>::v;
};
template <int B>
struct Pow<B, 0> {
  static constexpr int v = 1;
};

// ------------------------------------------------------------------------
// constant-bank tables (uploaded once per device and p)
// ------------------------------------------------------------------------
__constant__ double c_RC5[2][5][5], c_RS5[2][5][5], c_invD5[5];
__constant__ double c_RC7[2][7][7], c_RS7[2][7][7], c_invD7[7];
__constant__ double c_RC9[2][9][9], c_RS9[2][9][9], c_invD9[9];

template <int P>
struct CT;
template <>
struct CT<5> {
  __device__ __forceinline__ static double rc(int b, int m, int l) { return c_RC5[b][m][l]; }
  __device__ __forceinline__ static double rs(int b, int m, int l) { return c_RS5[b][m][l]; }
  __device__ __forceinline__ static double invD(int m) { return c_invD5[m]; }
};
template <>
struct CT<7> {
  __device__ __forceinline__ static double rc(int b, int m, int l) { return c_RC7[b][m][l]; }
  __device__ __forceinline__ static double rs(int b, int m, int l) { return c_RS7[b][m][l]; }
  __device__ __forceinline__ static double invD(int m) { return c_invD7[m]; }
};
template <>
struct CT<9> {
  __device__ __forceinline__ static double rc(int b, int m, int l) { return c_RC9[b][m][l]; }
  __device__ __forceinline__ static double rs(int b, int m, int l) { return c_RS9[b][m][l]; }
  __device__ __forceinline__ static double invD(int m) { return c_invD9[m]; }
};

cudaError_t upload_const_tables(int p, const double* RC, const double* RS, const double* invD) {
  const size_t n2 = sizeof(double) * 2 * p * p, n1 = sizeof(double) * p;
  cudaError_t e = cudaErrorInvalidValue;
  if (p == 5) {
    if ((e = cudaMemcpyToSymbol(c_RC5, RC, n2)) != cudaSuccess) return e;
    if ((e = cudaMemcpyToSymbol(c_RS5, RS, n2)) != cudaSuccess) return e;
    e = cudaMemcpyToSymbol(c_invD5, invD, n1);
  } else if (p == 7) {
    if ((e = cudaMemcpyToSymbol(c_RC7, RC, n2)) != cudaSuccess) return e;
    if ((e = cudaMemcpyToSymbol(c_RS7, RS, n2)) != cudaSuccess) return e;
    e = cudaMemcpyToSymbol(c_invD7, invD, n1);
  } else if (p == 9) {
    if ((e = cudaMemcpyToSymbol(c_RC9, RC, n2)) != cudaSuccess) return e;
    if ((e = cudaMemcpyToSymbol(c_RS9, RS, n2)) != cudaSuccess) return e;
    e = cudaMemcpyToSymbol(c_invD9, invD, n1);
  }
  return e;
}

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// ------------------------------------------------------------------------
// K2: leaf kernel, one warp per leaf B of T_K (h-representation)
// ------------------------------------------------------------------------
template <int D, int P>
__global__ __launch_bounds__(128) void k_leaf(const double* __restrict__ k_sorted, const int32_t* __restrict__ perm,
                                              const int32_t* __restrict__ first_pt,
                                              const double2* __restrict__ f, double2* __restrict__ out, int64_t b_lo,
                                              int64_t b_hi, int64_t N) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NACC = (PD + 31) / 32;
  constexpr int P1 = P - 1;
  __shared__ double r_s[4][D][P];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = b_lo + blockIdx.x * 4 + warp;
  if (b >= b_hi) return;
  double2 acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = make_double2(0.0, 0.0);
  const int j0 = first_pt[b], j1 = first_pt[b + 1];
  for (int j = j0; j < j1; ++j) {
    // s = k - c^B in [0,1] (exact); c^B = min(floor(k), N-1) per axis
    double ssum = 0.0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double kk = k_sorted[(int64_t)j * D + a];
      ssum += kk - fmin(floor(kk), (double)(N - 1));
    }
    if (lane < D * P) {
      const int a = lane / P, m = lane % P;
      const double kk = k_sorted[(int64_t)j * D + a];
      const double s = kk - fmin(floor(kk), (double)(N - 1));
      // r_m(s) = invD_m prod_{q != m} sin(pi (s P1 - q)/P1^2)
      double prod = CT<P>::invD(m);
#pragma unroll
      for (int q = 0; q < P; ++q)
        if (q != m) prod *= sinpi((s * P1 - q) / (double)(P1 * P1));
      r_s[warp][a][m] = prod;
    }
    __syncwarp();
    double sn, cs;
    sincospi(ssum, &sn, &cs);
    const double2 fj = cmul(f[perm[j]], make_double2(cs, sn));
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      const int e = lane + 32 * i;
      if (e < PD) {
        double w = 1.0;
        int r = e;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
          w *= r_s[warp][a][r % P];
          r /= P;
        }
        acc[i].x = fma(w, fj.x, acc[i].x);
        acc[i].y = fma(w, fj.y, acc[i].y);
      }
    }
    __syncwarp();
  }
  double2* o = out + (b - b_lo) * (int64_t)PD;
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    const int e = lane + 32 * i;
    if (e < PD) o[e] = acc[i];
  }
}

// ------------------------------------------------------------------------
// K3: translation kernel
// ------------------------------------------------------------------------
struct TransArgs {
  const double2* in;
  double2* out;
  const int32_t* cbK;
  const uint32_t* mK;
  const int32_t* cbX;
  const uint32_t* mX;
  int64_t b_lo, nAp_grp, ap_lo, ngroups;
  int64_t in_b0, in_nA, in_a0;
  int64_t out_b0, out_nA, out_a0;
  const int64_t* seg;  // [nseg+1] A boundaries at the output level, then [nseg] segment bases
  int nseg;
};

struct GroupMeta {
  int64_t iB, iAp;
  int32_t cbK, cbX;
  uint32_t mB, mA;
};

// projections of a child mask: set of top-k-bit prefixes / low-k-bit suffixes
template <int D>
__device__ __forceinline__ uint32_t proj_hi(uint32_t m, int k) {
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < (1 << D); ++c)
    if (m >> c & 1) r |= 1u << (c >> (D - k));
  return r;
}
template <int D>
__device__ __forceinline__ uint32_t proj_lo(uint32_t m, int k) {
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < (1 << D); ++c)
    if (m >> c & 1) r |= 1u << (c & ((1 << k) - 1));
  return r;
}
// index of the n-th set bit of m (n < popc(m))
__device__ __forceinline__ int nth_set(uint32_t m, int n) {
  for (int q = 0; q < n; ++q) m &= m - 1;
  return __ffs(m) - 1;
}

// One fiber, both outputs, children present per CLS (bit 0: beta=0, bit 1:
// beta=1); straight-line code over all rows so the compiler can interleave
// the independent DFMA chains.  CS form with constant-bank operands:
//   z_alpha[m] = sum_beta c_{alpha beta} (RC_beta[m] . x_beta + i (2 alpha - 1) RS_beta[m] . x_beta)
// c_{alpha,0} = 1, c_{0,1} = i, c_{1,1} = -i.
template <int P, int CLS, class Store>
__device__ __forceinline__ void contract_fiber(const double2 (&x0)[P], const double2 (&x1)[P], Store store) {
#pragma unroll
  for (int m = 0; m < P; ++m) {
    double2 z0 = make_double2(0.0, 0.0), z1 = make_double2(0.0, 0.0);
    if (CLS & 1) {
      double ur = 0.0, ui = 0.0, vr = 0.0, vi = 0.0;
#pragma unroll
      for (int l = 0; l < P; ++l) {
        const double c = CT<P>::rc(0, m, l), s = CT<P>::rs(0, m, l);
        ur = fma(c, x0[l].x, ur);
        ui = fma(c, x0[l].y, ui);
        vr = fma(s, x0[l].x, vr);
        vi = fma(s, x0[l].y, vi);
      }
      z0 = make_double2(ur + vi, ui - vr);
      z1 = make_double2(ur - vi, ui + vr);
    }
    if (CLS & 2) {
      double ur = 0.0, ui = 0.0, vr = 0.0, vi = 0.0;
#pragma unroll
      for (int l = 0; l < P; ++l) {
        const double c = CT<P>::rc(1, m, l), s = CT<P>::rs(1, m, l);
        ur = fma(c, x1[l].x, ur);
        ui = fma(c, x1[l].y, ui);
        vr = fma(s, x1[l].x, vr);
        vi = fma(s, x1[l].y, vi);
      }
      z0.x -= ui - vr;
      z0.y += ur + vi;
      z1.x += ui + vr;
      z1.y -= ur - vi;
    }
    store(m, z0, z1);
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// named barrier over the NT consumer threads (the producer warp never joins)
template <int NT>
__device__ __forceinline__ void cons_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
}

struct TaskEntry {
  uint8_t j, bp, as, cls;
};

// One axis pass over a tile of ng groups held in shared memory (slots
// [j][NS][PD]).  Tasks = (group, beta-prefix bp, alpha-suffix as) x fiber;
// each reads the fibers of slots (bp,0,as) and (bp,1,as) and writes both
// alpha outputs in place (or to HBM in the last pass).  Task entries are
// sorted by child class (both / beta=0 only / beta=1 only) so that warps run
// one straight-line code path.
template <int D, int P, int G, int NT, int AX, bool LAST, class Sync>
__device__ __forceinline__ void trans_pass(const TransArgs& a, double2* __restrict__ sb, const GroupMeta* gm, int ng,
                                           TaskEntry* ent, int* cnt, int tid, Sync sync) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NS = 1 << D;
  constexpr int PF = PD / P;
  constexpr int STR = Pow<P, D - 1 - AX>::v;  // stride of axis AX
  constexpr int SH = D - 1 - AX;              // bit of axis AX in a slot index
  constexpr int MAXE = G << (D - 1);  // combos per tile (upper bound)
  // cnt[0..2]: per-class counts (class 3, 1, 2); entries appended per class
  // (the order of independent tasks does not affect any result)
  if (tid < 3) cnt[tid] = 0;
  sync();
  if (tid < ng) {
    const uint32_t mB = gm[tid].mB, mA = gm[tid].mA;
    const uint32_t PBp = AX > 0 ? proj_hi<D>(mB, AX) : 1u;
    const uint32_t PAs = proj_lo<D>(mA, D - 1 - AX);
    const uint32_t PBa = proj_hi<D>(mB, AX + 1);
#pragma unroll
    for (int bp = 0; bp < (1 << AX); ++bp) {
      if (!(PBp >> bp & 1)) continue;
      const int cls = (int)((PBa >> (bp << 1)) & 3u);
      const int ci = cls == 3 ? 0 : (cls == 1 ? 1 : 2);
#pragma unroll
      for (int as = 0; as < (1 << (D - 1 - AX)); ++as) {
        if (!(PAs >> as & 1)) continue;
        const int pos = atomicAdd(&cnt[ci], 1);
        ent[ci * MAXE + pos] = TaskEntry{(uint8_t)tid, (uint8_t)bp, (uint8_t)as, (uint8_t)cls};
      }
    }
  }
  sync();
  const int n3 = cnt[0], n1 = cnt[1], n2 = cnt[2];
  const int ntot = (n3 + n1 + n2) * PF;
  for (int tau = tid; tau < ntot; tau += NT) {
    const int ei = tau / PF;
    const TaskEntry te = ei < n3 ? ent[ei] : (ei < n3 + n1 ? ent[MAXE + ei - n3] : ent[2 * MAXE + ei - n3 - n1]);
    const int f = tau % PF;
    const GroupMeta& g = gm[te.j];
    const int lo = f % STR, hi = f / STR;
    const int ebase = hi * STR * P + lo;
    const int slot0 = (te.bp << (D - AX)) | te.as;  // slot with bit SH = 0
    double2* s0 = sb + ((int64_t)te.j * NS + slot0) * PD + ebase;
    double2* s1 = sb + ((int64_t)te.j * NS + (slot0 | (1 << SH))) * PD + ebase;
    double2 x0[P], x1[P];
    double2* o0 = nullptr;
    double2* o1 = nullptr;
    if (!LAST) {
      o0 = s0;
      o1 = s1;
    } else {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int alpha = (t << SH) | te.as;  // child index of A within A'
        if (!(g.mA >> alpha & 1)) continue;
        const int64_t iA = (int64_t)g.cbX + __popc(g.mA & ((1u << alpha) - 1));
        int64_t pidx;
        if (a.nseg == 0) {
          pidx = (g.iB - a.out_b0) * a.out_nA + (iA - a.out_a0);
        } else {
          int q = 0;
          while (q + 1 < a.nseg && iA >= a.seg[q + 1]) ++q;
          const int64_t wq = a.seg[q + 1] - a.seg[q];
          pidx = a.seg[a.nseg + 1 + q] + (g.iB - a.out_b0) * wq + (iA - a.seg[q]);
        }
        (t ? o1 : o0) = a.out + pidx * PD + ebase;
      }
    }
    auto store = [&](int m, double2 z0, double2 z1) {
      if (o0) o0[m * STR] = z0;
      if (o1) o1[m * STR] = z1;
    };
#ifdef SFT_ABL_NOCOMPUTE
    if (true) {
#pragma unroll
      for (int m = 0; m < P; ++m) store(m, s0[m * STR], s1[m * STR]);
    } else
#endif
    if (te.cls == 3) {
#pragma unroll
      for (int l = 0; l < P; ++l) {
        x0[l] = s0[l * STR];
        x1[l] = s1[l * STR];
      }
      contract_fiber<P, 3>(x0, x1, store);
    } else if (te.cls == 1) {
#pragma unroll
      for (int l = 0; l < P; ++l) x0[l] = s0[l * STR];
      contract_fiber<P, 1>(x0, x1, store);
    } else {
#pragma unroll
      for (int l = 0; l < P; ++l) x1[l] = s1[l * STR];
      contract_fiber<P, 2>(x0, x1, store);
    }
  }
  sync();
}

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}

// Persistent, warp-specialised translation kernel.  Warp 0 is the producer:
// for each tile of G groups it reads the group metadata (child masks and
// first-child indices of B and A') and issues one 1-D TMA bulk copy per
// present child array into a 2-stage shared-memory ring (mbarrier
// complete_tx).  Warps 1..NT/32 consume: the axis passes run in place in the
// stage, the last pass stores the parent arrays to HBM, then the stage is
// released to the producer.  Loads of tile i+1 overlap the math of tile i.
template <int D, int P, int G, int NT, int NSTAGE>
__global__ __launch_bounds__(NT + 32, 1) void k_translate(TransArgs a, int64_t ntiles) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NS = 1 << D;
  constexpr int STAGE = G * NS * PD;  // double2 per stage
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* ring = reinterpret_cast<double2*>(smem_raw);  // [NSTAGE][G][NS][PD]
  __shared__ GroupMeta gm[NSTAGE][G];
  __shared__ int ngs[NSTAGE];
  __shared__ TaskEntry ent[3 * (G << (D - 1))];
  __shared__ int cnt[4];
  __shared__ __align__(8) uint64_t full[NSTAGE], empty[NSTAGE];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer ----------------
    for (int64_t i = 0;; ++i) {
      const int64_t tile = blockIdx.x + i * (int64_t)gridDim.x;
      if (tile >= ntiles) break;
      const int s = (int)(i % NSTAGE);
      if (i >= NSTAGE) mbar_wait(smem_u32(&empty[s]), (uint32_t)(((i / NSTAGE) + 1) & 1));
      const int64_t g0 = tile * G;
      const int ng = (int)min((int64_t)G, a.ngroups - g0);
      uint32_t nbytes = 0;
      if (lane < ng) {
        const int64_t g = g0 + lane;
        GroupMeta m;
        m.iB = a.b_lo + g / a.nAp_grp;
        m.iAp = a.ap_lo + g % a.nAp_grp;
        m.cbK = a.cbK[m.iB];
        m.mB = a.mK[m.iB];
        m.cbX = a.cbX[m.iAp];
        m.mA = a.mX[m.iAp];
        gm[s][lane] = m;
        nbytes = __popc(m.mB) * PD * (uint32_t)sizeof(double2);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) nbytes += __shfl_xor_sync(0xffffffffu, nbytes, o);
      if (lane == 0) {
        ngs[s] = ng;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                     "r"(nbytes)
                     : "memory");
      }
      __syncwarp();
      if (lane < ng) {
        const GroupMeta& m = gm[s][lane];
        uint32_t mm = m.mB;
        int r = 0;
        while (mm) {
          const int c = __ffs(mm) - 1;
          mm &= mm - 1;
          const int64_t iBc = (int64_t)m.cbK + r++;
          const int64_t pin = (iBc - a.in_b0) * a.in_nA + (m.iAp - a.in_a0);
          const double2* src = a.in + pin * PD;
          double2* dst = ring + (int64_t)s * STAGE + ((int64_t)lane * NS + c) * PD;
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  smem_u32(dst)),
              "l"(src), "r"((uint32_t)(PD * sizeof(double2))), "r"(smem_u32(&full[s]))
              : "memory");
        }
      }
    }
    return;
  }
  // ---------------- consumers ----------------
  const int tid = threadIdx.x - 32;
  for (int64_t i = 0;; ++i) {
    const int64_t tile = blockIdx.x + i * (int64_t)gridDim.x;
    if (tile >= ntiles) break;
    const int s = (int)(i % NSTAGE);
    mbar_wait(smem_u32(&full[s]), (uint32_t)((i / NSTAGE) & 1));
    double2* sb = ring + (int64_t)s * STAGE;
    const int ng = ngs[s];
    auto sync = [] { cons_sync<NT>(); };
    if constexpr (D == 2) {
      trans_pass<D, P, G, NT, 1, false>(a, sb, gm[s], ng, ent, cnt, tid, sync);
      trans_pass<D, P, G, NT, 0, true>(a, sb, gm[s], ng, ent, cnt, tid, sync);
    } else {
      trans_pass<D, P, G, NT, 2, false>(a, sb, gm[s], ng, ent, cnt, tid, sync);
      trans_pass<D, P, G, NT, 1, false>(a, sb, gm[s], ng, ent, cnt, tid, sync);
      trans_pass<D, P, G, NT, 0, true>(a, sb, gm[s], ng, ent, cnt, tid, sync);
    }
    if (tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
  }
}

// Non-persistent variant: one CTA per tile, single stage; several CTAs per SM
// overlap loads and math.  Selected per (d, p) by TransCfg::PERSIST.
#ifdef SFT_INSTR
__device__ unsigned long long* g_instr = nullptr;  // [blocks][8]
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define INSTR(k)                                                        \
  if (threadIdx.x == 0 && g_instr) g_instr[(size_t)blockIdx.x * 8 + (k)] = gtime();
#else
#define INSTR(k)
#endif

// minBlocksPerSM: target 16 resident warps (an explicit 1 lets ptxas take
// ~200 registers and halves occupancy; forcing fewer than ~120 spills)
#ifndef SFT_WARPS_PER_SM
#define SFT_WARPS_PER_SM 16
#endif
#define SFT_MINB(NT) ((SFT_WARPS_PER_SM * 32 / (NT)) > 0 ? (SFT_WARPS_PER_SM * 32 / (NT)) : 1)
template <int D, int P, int G, int NT>
__global__ __launch_bounds__(NT, SFT_MINB(NT)) void k_translate_np(TransArgs a) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NS = 1 << D;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* sb = reinterpret_cast<double2*>(smem_raw);  // [G][NS][PD]
  __shared__ GroupMeta gm[G];
  __shared__ TaskEntry ent[3 * (G << (D - 1))];
  __shared__ int cnt[4];
  __shared__ __align__(8) uint64_t bar;
  INSTR(0);
  const int64_t g0 = (int64_t)blockIdx.x * G;
  const int ng = (int)min((int64_t)G, a.ngroups - g0);
  if (threadIdx.x < ng) {
    const int64_t g = g0 + threadIdx.x;
    GroupMeta m;
    m.iB = a.b_lo + g / a.nAp_grp;
    m.iAp = a.ap_lo + g % a.nAp_grp;
    m.cbK = a.cbK[m.iB];
    m.mB = a.mK[m.iB];
    m.cbX = a.cbX[m.iAp];
    m.mA = a.mX[m.iAp];
    gm[threadIdx.x] = m;
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    uint32_t nbytes = lane < ng ? __popc(gm[lane].mB) * PD * (uint32_t)sizeof(double2) : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) nbytes += __shfl_xor_sync(0xffffffffu, nbytes, o);
    if (lane == 0)
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(nbytes)
                   : "memory");
    __syncwarp();
    if (lane < ng) {
      const GroupMeta& m = gm[lane];
      uint32_t mm = m.mB;
      int r = 0;
      while (mm) {
        const int c = __ffs(mm) - 1;
        mm &= mm - 1;
        const int64_t iBc = (int64_t)m.cbK + r++;
        const int64_t pin = (iBc - a.in_b0) * a.in_nA + (m.iAp - a.in_a0);
#ifndef SFT_ABL_NOLOAD
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(sb + ((int64_t)lane * NS + c) * PD)),
            "l"(a.in + pin * PD), "r"((uint32_t)(PD * sizeof(double2))), "r"(smem_u32(&bar))
            : "memory");
#else
        (void)pin;
        asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)),
                     "r"((uint32_t)(PD * sizeof(double2))) : "memory");
#endif
      }
    }
  }
  INSTR(1);
  mbar_wait(smem_u32(&bar), 0);
  INSTR(2);
  auto sync = [] { __syncthreads(); };
  const int tid = threadIdx.x;
  if constexpr (D == 2) {
    trans_pass<D, P, G, NT, 1, false>(a, sb, gm, ng, ent, cnt, tid, sync);
    INSTR(3);
    trans_pass<D, P, G, NT, 0, true>(a, sb, gm, ng, ent, cnt, tid, sync);
    INSTR(4);
#ifdef SFT_INSTR
    if (threadIdx.x == 0 && g_instr) {
      unsigned smid;
      asm("mov.u32 %0, %smid;" : "=r"(smid));
      g_instr[(size_t)blockIdx.x * 8 + 7] = smid;
    }
#endif
  } else {
    trans_pass<D, P, G, NT, 2, false>(a, sb, gm, ng, ent, cnt, tid, sync);
    trans_pass<D, P, G, NT, 1, false>(a, sb, gm, ng, ent, cnt, tid, sync);
    trans_pass<D, P, G, NT, 0, true>(a, sb, gm, ng, ent, cnt, tid, sync);
  }
}

// ------------------------------------------------------------------------
// K4: final kernel, one warp per leaf A of T_X (h-representation)
// ------------------------------------------------------------------------
template <int D, int P>
__global__ __launch_bounds__(128) void k_final(const double* __restrict__ x_sorted, const int32_t* __restrict__ perm,
                                               const int32_t* __restrict__ first_pt,
                                               const double2* __restrict__ h0, double2* __restrict__ u,
                                               int64_t a_lo, int64_t a_hi, int64_t N) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NACC = (PD + 31) / 32;
  constexpr int P1 = P - 1;
  __shared__ double2 e_s[4][D][P];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t A = a_lo + blockIdx.x * 4 + warp;
  if (A >= a_hi) return;
  const double2* h = h0 + (A - a_lo) * (int64_t)PD;
  double2 hr[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    const int e = lane + 32 * i;
    hr[i] = e < PD ? h[e] : make_double2(0.0, 0.0);
  }
  const int j0 = first_pt[A], j1 = first_pt[A + 1];
  for (int j = j0; j < j1; ++j) {
    if (lane < D * P) {
      const int a = lane / P, l = lane % P;
      const double xx = x_sorted[(int64_t)j * D + a];
      const double xi = xx - fmin(floor(xx), (double)(N - 1));  // in [0,1], exact
      double sn, cs;
      sincospi((2.0 * xi - 1.0) * l / P1, &sn, &cs);
      e_s[warp][a][l] = make_double2(cs, sn);
    }
    __syncwarp();
    double2 s = make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      const int e = lane + 32 * i;
      if (e < PD) {
        double2 w = hr[i];
        int r = e;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
          w = cmul(w, e_s[warp][a][r % P]);
          r /= P;
        }
        s.x += w.x;
        s.y += w.y;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      s.x += __shfl_xor_sync(0xffffffffu, s.x, o);
      s.y += __shfl_xor_sync(0xffffffffu, s.y, o);
    }
    if (lane == 0) u[perm[j]] = s;
    __syncwarp();
  }
}

__global__ void k_zero(double2* p, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = make_double2(0.0, 0.0);
}

// ------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------
// tile configuration: G groups per CTA, NT threads (tuned on B200)
#ifndef SFT_PERSIST
#define SFT_PERSIST 0
#endif
#ifndef SFT_NSTAGE
#define SFT_NSTAGE 2
#endif
#ifndef SFT_G25
#define SFT_G25 16
#define SFT_NT25 128
#endif
#ifndef SFT_G27
#define SFT_G27 12
#define SFT_NT27 128
#endif
#ifndef SFT_G29
#define SFT_G29 16
#define SFT_NT29 256
#endif
#ifndef SFT_G35
#define SFT_G35 4
#define SFT_NT35 256
#endif
#ifndef SFT_G37
#define SFT_G37 2
#define SFT_NT37 256
#endif
#ifndef SFT_G39
#define SFT_G39 1
#define SFT_NT39 256
#endif
template <int D, int P>
struct TransCfg;
template <>
struct TransCfg<2, 5> { static constexpr int G = SFT_G25, NT = SFT_NT25, PERSIST = SFT_PERSIST; };
template <>
struct TransCfg<2, 7> { static constexpr int G = SFT_G27, NT = SFT_NT27, PERSIST = SFT_PERSIST; };
template <>
struct TransCfg<2, 9> { static constexpr int G = SFT_G29, NT = SFT_NT29, PERSIST = SFT_PERSIST; };
template <>
struct TransCfg<3, 5> { static constexpr int G = SFT_G35, NT = SFT_NT35, PERSIST = SFT_PERSIST; };
template <>
struct TransCfg<3, 7> { static constexpr int G = SFT_G37, NT = SFT_NT37, PERSIST = SFT_PERSIST; };
template <>
struct TransCfg<3, 9> { static constexpr int G = SFT_G39, NT = SFT_NT39, PERSIST = SFT_PERSIST; };

template <int D, int P>
static cudaError_t launch_translate_t(const sft_plan_s* Pl, const LevelDims& L, const double2* in, double2* out) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int G = TransCfg<D, P>::G, NT = TransCfg<D, P>::NT;
  constexpr bool PERSIST = TransCfg<D, P>::PERSIST != 0;
  constexpr int NSTAGE = SFT_NSTAGE;
  const size_t smem = (size_t)(PERSIST ? NSTAGE : 1) * G * (1 << D) * PD * sizeof(double2);
  static int blocks_per_sm = -1, nsm = 0;
  if (blocks_per_sm < 0) {
    cudaError_t e = PERSIST ? cudaFuncSetAttribute(k_translate<D, P, G, NT, NSTAGE>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                            : cudaFuncSetAttribute(k_translate_np<D, P, G, NT>,
                                                   cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = PERSIST ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_translate<D, P, G, NT, NSTAGE>, NT + 32, smem)
                : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_translate_np<D, P, G, NT>, NT, smem);
    if (e != cudaSuccess) return e;
    if (blocks_per_sm < 1) return cudaErrorInvalidConfiguration;
  }
  TransArgs a;
  a.in = in;
  a.out = out;
  a.cbK = L.cbK;
  a.mK = L.mK;
  a.cbX = L.cbX;
  a.mX = L.mX;
  a.b_lo = L.b_lo;
  a.nAp_grp = L.ap_hi - L.ap_lo;
  a.ap_lo = L.ap_lo;
  a.ngroups = (L.b_hi - L.b_lo) * a.nAp_grp;
  a.in_b0 = L.in_b0;
  a.in_nA = L.in_nA;
  a.in_a0 = L.in_a0;
  a.out_b0 = L.out_b0;
  a.out_nA = L.out_nA;
  a.out_a0 = L.out_a0;
  a.seg = L.seg;
  a.nseg = L.nseg;
  if (a.ngroups <= 0) return cudaSuccess;
  const int64_t ntiles = (a.ngroups + G - 1) / G;
  if (PERSIST) {
    const int64_t grid = std::min<int64_t>(ntiles, (int64_t)nsm * blocks_per_sm);
    k_translate<D, P, G, NT, NSTAGE><<<(unsigned)grid, NT + 32, smem, Pl->stream>>>(a, ntiles);
  } else {
    k_translate_np<D, P, G, NT><<<(unsigned)ntiles, NT, smem, Pl->stream>>>(a);
  }
  count_launch();
  return cudaGetLastError();
}

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

cudaError_t launch_translate(const sft_plan_s* Pl, const LevelDims& L, const double2* in, double2* out) {
  SFT_DISPATCH(Pl->d, Pl->p, return (launch_translate_t<D, P>(Pl, L, in, out)));
  return cudaSuccess;
}

cudaError_t launch_leaf(const sft_plan_s* Pl, const double2* f, double2* out, int64_t b_lo, int64_t b_hi) {
  if (b_hi <= b_lo) return cudaSuccess;
  const unsigned nb = (unsigned)((b_hi - b_lo + 3) / 4);
  SFT_DISPATCH(Pl->d, Pl->p,
               (k_leaf<D, P><<<nb, 128, 0, Pl->stream>>>(Pl->K.pts_sorted, Pl->K.perm, Pl->K.first_pt, f, out, b_lo,
                                                         b_hi, Pl->N)));
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_final(const sft_plan_s* Pl, const double2* h0, double2* u, int64_t a_lo, int64_t a_hi) {
  if (a_hi <= a_lo) return cudaSuccess;
  const unsigned nb = (unsigned)((a_hi - a_lo + 3) / 4);
  SFT_DISPATCH(Pl->d, Pl->p,
               (k_final<D, P><<<nb, 128, 0, Pl->stream>>>(Pl->X.pts_sorted, Pl->X.perm, Pl->X.first_pt, h0, u, a_lo,
                                                          a_hi, Pl->N)));
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_zero(double2* p, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_zero<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, n);
  count_launch();
  return cudaGetLastError();
}

}  // namespace sft

#ifdef SFT_INSTR
extern "C" int sft_instr_set(void* dev_buf) {
  return cudaMemcpyToSymbol(sft::g_instr, &dev_buf, sizeof(void*)) == cudaSuccess ? 0 : 4;
}
#endif

extern "C" int sft_launch_count(int64_t* out) {
  if (!out) return SFT_E_ARG;
  *out = (int64_t)sft::launch_count();
  return SFT_OK;
}
