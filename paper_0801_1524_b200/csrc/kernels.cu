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

// y_alpha += T[alpha][B] x  for both alpha (CS form, constant-bank operands)
template <int P, int B>
__device__ __forceinline__ void contract(const double2 (&x)[P], double2 (&z0)[P], double2 (&z1)[P]) {
#pragma unroll
  for (int m = 0; m < P; ++m) {
    double ur = 0.0, ui = 0.0, vr = 0.0, vi = 0.0;
#pragma unroll
    for (int l = 0; l < P; ++l) {
      const double c = CT<P>::rc(B, m, l), s = CT<P>::rs(B, m, l);
      ur = fma(c, x[l].x, ur);
      ui = fma(c, x[l].y, ui);
      vr = fma(s, x[l].x, vr);
      vi = fma(s, x[l].y, vi);
    }
    // alpha=0: u - i v = (ur + vi) + i (ui - vr);  alpha=1: u + i v = (ur - vi) + i (ui + vr)
    if (B == 0) {
      z0[m].x += ur + vi;
      z0[m].y += ui - vr;
      z1[m].x += ur - vi;
      z1[m].y += ui + vr;
    } else {  // c_{0,1} = i, c_{1,1} = -i
      z0[m].x -= ui - vr;
      z0[m].y += ur + vi;
      z1[m].x += ui + vr;
      z1[m].y -= ur - vi;
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int D, int P, int G, int NT, int AX, bool LAST>
__device__ __forceinline__ void trans_pass(const TransArgs& a, double2* __restrict__ sb, const GroupMeta* gm, int ng,
                                           int* pre) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NS = 1 << D;
  constexpr int PF = PD / P;
  constexpr int STR = Pow<P, D - 1 - AX>::v;  // stride of axis AX
  constexpr int SH = D - 1 - AX;              // bit of axis AX in a slot index
  // per-group task counts -> prefix (G is small)
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int j = 0; j < ng; ++j) {
      pre[j] = acc;
      const uint32_t PBp = AX > 0 ? proj_hi<D>(gm[j].mB, AX) : 1u;
      const uint32_t PAs = proj_lo<D>(gm[j].mA, D - 1 - AX);
      acc += __popc(PBp) * __popc(PAs) * PF;
    }
    pre[ng] = acc;
  }
  __syncthreads();
  const int ntot = pre[ng];
  for (int tau = threadIdx.x; tau < ntot; tau += NT) {
    int j = 0;
    while (j + 1 < ng && tau >= pre[j + 1]) ++j;
    const GroupMeta g = gm[j];
    const int local = tau - pre[j];
    const int combo = local / PF, f = local % PF;
    const uint32_t PBp = AX > 0 ? proj_hi<D>(g.mB, AX) : 1u;
    const uint32_t PAs = proj_lo<D>(g.mA, D - 1 - AX);
    const uint32_t PBa = proj_hi<D>(g.mB, AX + 1);
    const uint32_t PAa = proj_lo<D>(g.mA, D - AX);
    const int nas = __popc(PAs);
    const int bp = nth_set(PBp, combo / nas), as = nth_set(PAs, combo % nas);
    const bool vb0 = PBa >> (bp << 1) & 1, vb1 = PBa >> ((bp << 1) | 1) & 1;
    const int lo = f % STR, hi = f / STR;
    const int ebase = hi * STR * P + lo;
    const int slot0 = (bp << (D - AX)) | as;  // slot with bit SH = 0
    double2* s0 = sb + ((int64_t)j * NS + slot0) * PD + ebase;
    double2* s1 = sb + ((int64_t)j * NS + (slot0 | (1 << SH))) * PD + ebase;
    double2 z0[P], z1[P], x[P];
#pragma unroll
    for (int m = 0; m < P; ++m) z0[m] = z1[m] = make_double2(0.0, 0.0);
    if (vb0) {
#pragma unroll
      for (int l = 0; l < P; ++l) x[l] = s0[l * STR];
      contract<P, 0>(x, z0, z1);
    }
    if (vb1) {
#pragma unroll
      for (int l = 0; l < P; ++l) x[l] = s1[l * STR];
      contract<P, 1>(x, z0, z1);
    }
    if (!LAST) {
      // in place: slot (bp, t, as) now holds alpha_AX = t
#pragma unroll
      for (int m = 0; m < P; ++m) {
        s0[m * STR] = z0[m];
        s1[m * STR] = z1[m];
      }
    } else {
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        const int alpha = (t << SH) | as;  // child index of A within A'
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
        double2* o = a.out + pidx * PD + ebase;
        const double2* z = t ? z1 : z0;
#pragma unroll
        for (int m = 0; m < P; ++m) o[m * STR] = z[m];
      }
    }
  }
  __syncthreads();
}

template <int D, int P, int G, int NT>
__global__ __launch_bounds__(NT) void k_translate(TransArgs a) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NS = 1 << D;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  double2* sb = reinterpret_cast<double2*>(smem_raw);  // [G][NS][PD]
  __shared__ GroupMeta gm[G];
  __shared__ int pre[G + 1];
  __shared__ __align__(8) uint64_t bar;

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
  // stage the child arrays h^{A' B_c} of every group into slot c with 1-D TMA
  if (threadIdx.x == 0) {
    uint32_t bytes = 0;
    for (int j = 0; j < ng; ++j) bytes += __popc(gm[j].mB) * PD * (uint32_t)sizeof(double2);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes)
                 : "memory");
    for (int j = 0; j < ng; ++j) {
      uint32_t mm = gm[j].mB;
      int r = 0;
      while (mm) {
        const int c = __ffs(mm) - 1;
        mm &= mm - 1;
        const int64_t iBc = (int64_t)gm[j].cbK + r++;
        const int64_t pin = (iBc - a.in_b0) * a.in_nA + (gm[j].iAp - a.in_a0);
        const double2* src = a.in + pin * PD;
        double2* dst = sb + ((int64_t)j * NS + c) * PD;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(dst)),
            "l"(src), "r"((uint32_t)(PD * sizeof(double2))), "r"(smem_u32(&bar))
            : "memory");
      }
    }
  }
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
          : "=r"(done)
          : "r"(smem_u32(&bar))
          : "memory");
    }
  }
  if constexpr (D == 2) {
    trans_pass<D, P, G, NT, 1, false>(a, sb, gm, ng, pre);
    trans_pass<D, P, G, NT, 0, true>(a, sb, gm, ng, pre);
  } else {
    trans_pass<D, P, G, NT, 2, false>(a, sb, gm, ng, pre);
    trans_pass<D, P, G, NT, 1, false>(a, sb, gm, ng, pre);
    trans_pass<D, P, G, NT, 0, true>(a, sb, gm, ng, pre);
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
template <int D, int P>
struct TransCfg;
template <>
struct TransCfg<2, 5> { static constexpr int G = 16, NT = 128; };
template <>
struct TransCfg<2, 7> { static constexpr int G = 12, NT = 128; };
template <>
struct TransCfg<2, 9> { static constexpr int G = 8, NT = 128; };
template <>
struct TransCfg<3, 5> { static constexpr int G = 4, NT = 256; };
template <>
struct TransCfg<3, 7> { static constexpr int G = 2, NT = 256; };
template <>
struct TransCfg<3, 9> { static constexpr int G = 1, NT = 256; };

template <int D, int P>
static cudaError_t launch_translate_t(const sft_plan_s* Pl, const LevelDims& L, const double2* in, double2* out) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int G = TransCfg<D, P>::G, NT = TransCfg<D, P>::NT;
  const size_t smem = (size_t)G * (1 << D) * PD * sizeof(double2);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_translate<D, P, G, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    attr_set = true;
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
  const int64_t nblocks = (a.ngroups + G - 1) / G;
  k_translate<D, P, G, NT><<<(unsigned)nblocks, NT, smem, Pl->stream>>>(a);
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

extern "C" int sft_launch_count(int64_t* out) {
  if (!out) return SFT_E_ARG;
  *out = (int64_t)sft::launch_count();
  return SFT_OK;
}
