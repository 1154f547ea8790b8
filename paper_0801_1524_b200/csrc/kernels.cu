// kernels.cu -- steps 2-4 of the butterfly as sm_100a
// FP64 kernels in the box-relative formulation (sft_internal.cuh).
//
//   K2 leaf:        g^{A0 B}_m = sum_{k_j in B} f_j  prod_ax w_{m_ax}(k_j,ax - c^B_ax)
//   K3 translation: g^{AB} = sum_{present B_c} (x)_ax V[alpha_ax][beta_ax] g^{A' B_c}
//                   one CTA = GPC groups (A', B); each group reads <= 2^d child
//                   arrays, writes <= 2^d parent arrays; sum-factorised axis by
//                   axis through shared memory, masks drive which slots exist.
//   K4 final:       u_i = sum_l prod_ax e^{2 pi i (x_i - c^A) l_ax/(p-1)} g^{A B0}_l
//
// Numerics: no G^{-1} anywhere; leaf weights by the sine-product form of the
// Lagrange basis (small arguments of sinpi/cospi only).  No floating-point
// atomics: every output is written by exactly one thread in a fixed order,
// so results are bitwise reproducible.
#include "sft_internal.cuh"

namespace sft {

template <int B, int E>
struct Pow {
  static constexpr int v = B * Pow<B, E - 1>::v;
};
template <int B>
struct Pow<B, 0> {
  static constexpr int v = 1;
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ void cfma(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}

// ------------------------------------------------------------------------
// K2: leaf kernel, one warp per leaf B of T_K
// ------------------------------------------------------------------------
template <int D, int P>
__global__ __launch_bounds__(128) void k_leaf(const double* __restrict__ k_sorted, const int32_t* __restrict__ perm,
                                              const int32_t* __restrict__ first_pt,
                                              const double2* __restrict__ f, const double* __restrict__ invD,
                                              double2* __restrict__ out, int64_t b_lo, int64_t b_hi, int64_t N) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NACC = (PD + 31) / 32;
  constexpr int P1 = P - 1;
  __shared__ double2 w_s[4][D][P];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t b = b_lo + blockIdx.x * 4 + warp;
  if (b >= b_hi) return;
  double2 acc[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) acc[i] = make_double2(0.0, 0.0);
  const int j0 = first_pt[b], j1 = first_pt[b + 1];
  // leaf corner from any point of the leaf
  double cB[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    double c = floor(k_sorted[(int64_t)j0 * D + a]);
    cB[a] = fmin(c, (double)(N - 1));
  }
  for (int j = j0; j < j1; ++j) {
    if (lane < D * P) {
      const int a = lane / P, m = lane % P;
      const double s = k_sorted[(int64_t)j * D + a] - cB[a];  // in [0,1], exact
      // prod_{q != m} sin(pi (s P1 - q) / P1^2)
      double prod = 1.0;
#pragma unroll
      for (int q = 0; q < P; ++q)
        if (q != m) prod *= sinpi((s * P1 - q) / (double)(P1 * P1));
      double sn, cs;
      sincospi(s - (double)m / P1, &sn, &cs);
      prod *= invD[m];
      w_s[warp][a][m] = make_double2(prod * cs, prod * sn);
    }
    __syncwarp();
    const double2 fj = f[perm[j]];
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      const int e = lane + 32 * i;
      if (e < PD) {
        double2 w = fj;
        int r = e;
#pragma unroll
        for (int a = D - 1; a >= 0; --a) {
          w = cmul(w, w_s[warp][a][r % P]);
          r /= P;
        }
        acc[i].x += w.x;
        acc[i].y += w.y;
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
struct GroupMeta {
  int64_t iB, iAp;
  int32_t cbK, cbX;
  uint32_t mB, mA;
  int valid;
};
struct TaskEntry {
  uint8_t j, bpre, asuf, vb, va;
};

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
  const double2* V;
};

// projection masks: PB(mB, k) = set of top-k-bit prefixes (as k-bit values) of
// the present child indices; PA(mA, k) = set of low-k-bit suffixes.
template <int D>
__device__ __forceinline__ uint32_t proj_hi(uint32_t m, int k) {
  uint32_t r = 0;
  for (int c = 0; c < (1 << D); ++c)
    if (m >> c & 1) r |= 1u << (c >> (D - k));
  return r;
}
template <int D>
__device__ __forceinline__ uint32_t proj_lo(uint32_t m, int k) {
  uint32_t r = 0;
  for (int c = 0; c < (1 << D); ++c)
    if (m >> c & 1) r |= 1u << (c & ((1 << k) - 1));
  return r;
}

template <int D, int P, int AX, int GPC, int NT, bool LAST>
__device__ __forceinline__ void trans_pass(const TransArgs& a, const double2* __restrict__ sV,
                                           const double2* __restrict__ src, double2* __restrict__ dst,
                                           const GroupMeta* gm, TaskEntry* tasks, int* ntask) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NS = 1 << D;
  constexpr int PF = PD / P;
  constexpr int STR = Pow<P, D - 1 - AX>::v;  // stride of axis AX
  if (threadIdx.x == 0) {
    int nt = 0;
    for (int j = 0; j < GPC; ++j) {
      if (!gm[j].valid) continue;
      const uint32_t mB = gm[j].mB, mA = gm[j].mA;
      const uint32_t PBa = proj_hi<D>(mB, AX + 1);       // (AX+1)-bit beta prefixes incl. beta_AX
      const uint32_t PBp = AX > 0 ? proj_hi<D>(mB, AX) : 1u;  // AX-bit prefixes
      const uint32_t PAs = proj_lo<D>(mA, D - 1 - AX);   // alpha suffix (axes > AX)
      const uint32_t PAa = proj_lo<D>(mA, D - AX);       // alpha suffix incl. alpha_AX
      for (int bp = 0; bp < (1 << AX); ++bp) {
        if (!(PBp >> bp & 1)) continue;
        for (int as = 0; as < (1 << (D - 1 - AX)); ++as) {
          if (!(PAs >> as & 1)) continue;
          uint8_t vb = 0, va = 0;
          for (int t = 0; t < 2; ++t) {
            if (PBa >> ((bp << 1) | t) & 1) vb |= 1 << t;
            if (PAa >> ((t << (D - 1 - AX)) | as) & 1) va |= 1 << t;
          }
          tasks[nt++] = TaskEntry{(uint8_t)j, (uint8_t)bp, (uint8_t)as, vb, va};
        }
      }
    }
    *ntask = nt;
  }
  __syncthreads();
  const int ntot = *ntask * PF;
  for (int tau = threadIdx.x; tau < ntot; tau += NT) {
    const TaskEntry te = tasks[tau / PF];
    const int f = tau % PF;
    const int lo = f % STR, hi = f / STR;
    const int ebase = hi * STR * P + lo;
    const int shift = D - 1 - AX;
    double2 x[2][P];
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int slot = (te.bpre << (D - AX)) | (t << shift) | te.asuf;
      const double2* s = src + ((int64_t)te.j * NS + slot) * PD + ebase;
      if (te.vb >> t & 1) {
#pragma unroll
        for (int l = 0; l < P; ++l) x[t][l] = s[l * STR];
      } else {
#pragma unroll
        for (int l = 0; l < P; ++l) x[t][l] = make_double2(0.0, 0.0);
      }
    }
#pragma unroll
    for (int al = 0; al < 2; ++al) {
      if (!(te.va >> al & 1)) continue;
      double2 y[P];
#pragma unroll
      for (int m = 0; m < P; ++m) y[m] = make_double2(0.0, 0.0);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (!(te.vb >> t & 1)) continue;
        const double2* Vt = sV + (al * 2 + t) * P * P;
#pragma unroll
        for (int m = 0; m < P; ++m) {
#pragma unroll
          for (int l = 0; l < P; ++l) cfma(y[m], Vt[m * P + l], x[t][l]);
        }
      }
      const int oslot = (te.bpre << (D - AX)) | (al << shift) | te.asuf;
      if (!LAST) {
        double2* o = dst + ((int64_t)te.j * NS + oslot) * PD + ebase;
#pragma unroll
        for (int m = 0; m < P; ++m) o[m * STR] = y[m];
      } else {
        // AX == 0: oslot is the child index alpha of A within A'
        const GroupMeta& g = gm[te.j];
        const int rank = __popc(g.mA & ((1u << oslot) - 1));
        const int64_t iA = (int64_t)g.cbX + rank;
        int64_t pidx;
        if (a.nseg == 0) {
          pidx = (g.iB - a.out_b0) * a.out_nA + (iA - a.out_a0);
        } else {
          int q = 0;
          while (q + 1 < a.nseg && iA >= a.seg[q + 1]) ++q;
          const int64_t w = a.seg[q + 1] - a.seg[q];
          pidx = a.seg[a.nseg + 1 + q] + (g.iB - a.out_b0) * w + (iA - a.seg[q]);
        }
        double2* o = a.out + pidx * PD + ebase;
#pragma unroll
        for (int m = 0; m < P; ++m) o[m * STR] = y[m];
      }
    }
  }
  __syncthreads();
}

template <int D, int P, int GPC, int NT>
__global__ __launch_bounds__(NT) void k_translate(TransArgs a) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NS = 1 << D;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double2* sV = reinterpret_cast<double2*>(smem_raw);
  double2* bufA = sV + 4 * P * P;
  double2* bufB = bufA + GPC * NS * PD;
  __shared__ GroupMeta gm[GPC];
  __shared__ TaskEntry tasks[GPC * NS];
  __shared__ int ntask;

  for (int i = threadIdx.x; i < 4 * P * P; i += NT) sV[i] = a.V[i];
  const int64_t g0 = (int64_t)blockIdx.x * GPC;
  if (threadIdx.x < GPC) {
    const int64_t g = g0 + threadIdx.x;
    GroupMeta m;
    m.valid = g < a.ngroups;
    if (m.valid) {
      m.iB = a.b_lo + g / a.nAp_grp;
      m.iAp = a.ap_lo + g % a.nAp_grp;
      m.cbK = a.cbK[m.iB];
      m.mB = a.mK[m.iB];
      m.cbX = a.cbX[m.iAp];
      m.mA = a.mX[m.iAp];
    } else {
      m.iB = m.iAp = 0;
      m.cbK = m.cbX = 0;
      m.mB = m.mA = 0;
    }
    gm[threadIdx.x] = m;
  }
  __syncthreads();
  // stage child arrays g^{A' B_c} into slot beta = c of each group
  for (int j = 0; j < GPC; ++j) {
    if (!gm[j].valid) continue;
    const uint32_t mB = gm[j].mB;
    const int nch = __popc(mB);
    for (int idx = threadIdx.x; idx < nch * PD; idx += NT) {
      const int r = idx / PD, e = idx % PD;
      // r-th present child
      uint32_t mm = mB;
      for (int q = 0; q < r; ++q) mm &= mm - 1;
      const int c = __ffs(mm) - 1;
      const int64_t iBc = (int64_t)gm[j].cbK + r;
      const int64_t pin = (iBc - a.in_b0) * a.in_nA + (gm[j].iAp - a.in_a0);
      bufA[((int64_t)j * NS + c) * PD + e] = a.in[pin * PD + e];
    }
  }
  __syncthreads();
  if constexpr (D == 2) {
    trans_pass<D, P, 1, GPC, NT, false>(a, sV, bufA, bufB, gm, tasks, &ntask);
    trans_pass<D, P, 0, GPC, NT, true>(a, sV, bufB, nullptr, gm, tasks, &ntask);
  } else {
    trans_pass<D, P, 2, GPC, NT, false>(a, sV, bufA, bufB, gm, tasks, &ntask);
    trans_pass<D, P, 1, GPC, NT, false>(a, sV, bufB, bufA, gm, tasks, &ntask);
    trans_pass<D, P, 0, GPC, NT, true>(a, sV, bufA, nullptr, gm, tasks, &ntask);
  }
}

// ------------------------------------------------------------------------
// K4: final kernel, one warp per leaf A of T_X
// ------------------------------------------------------------------------
template <int D, int P>
__global__ __launch_bounds__(128) void k_final(const double* __restrict__ x_sorted, const int32_t* __restrict__ perm,
                                               const int32_t* __restrict__ first_pt,
                                               const double2* __restrict__ g0, double2* __restrict__ u,
                                               int64_t a_lo, int64_t a_hi, int64_t N) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NACC = (PD + 31) / 32;
  constexpr int P1 = P - 1;
  __shared__ double2 e_s[4][D][P];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t A = a_lo + blockIdx.x * 4 + warp;
  if (A >= a_hi) return;
  const double2* g = g0 + (A - a_lo) * (int64_t)PD;
  double2 gr[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    const int e = lane + 32 * i;
    gr[i] = e < PD ? g[e] : make_double2(0.0, 0.0);
  }
  const int j0 = first_pt[A], j1 = first_pt[A + 1];
  double cA[D];
#pragma unroll
  for (int a = 0; a < D; ++a) cA[a] = fmin(floor(x_sorted[(int64_t)j0 * D + a]), (double)(N - 1));
  for (int j = j0; j < j1; ++j) {
    if (lane < D * P) {
      const int a = lane / P, l = lane % P;
      const double xi = x_sorted[(int64_t)j * D + a] - cA[a];  // in [0,1], exact
      double sn, cs;
      sincospi(2.0 * xi * l / P1, &sn, &cs);
      e_s[warp][a][l] = make_double2(cs, sn);
    }
    __syncwarp();
    double2 s = make_double2(0.0, 0.0);
#pragma unroll
    for (int i = 0; i < NACC; ++i) {
      const int e = lane + 32 * i;
      if (e < PD) {
        double2 w = gr[i];
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
struct TransCfg<2, 5> { static constexpr int GPC = 8, NT = 128; };
template <>
struct TransCfg<2, 7> { static constexpr int GPC = 8, NT = 128; };
template <>
struct TransCfg<2, 9> { static constexpr int GPC = 8, NT = 128; };
template <>
struct TransCfg<3, 5> { static constexpr int GPC = 2, NT = 128; };
template <>
struct TransCfg<3, 7> { static constexpr int GPC = 1, NT = 128; };
template <>
struct TransCfg<3, 9> { static constexpr int GPC = 1, NT = 256; };

template <int D, int P>
static cudaError_t launch_translate_t(const sft_plan_s* Pl, const LevelDims& L, const double2* in, double2* out) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int GPC = TransCfg<D, P>::GPC, NT = TransCfg<D, P>::NT;
  const size_t smem = (size_t)(4 * P * P + 2 * GPC * (1 << D) * PD) * sizeof(double2);
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_translate<D, P, GPC, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
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
  a.V = Pl->tab->V;
  if (a.ngroups <= 0) return cudaSuccess;
  const int64_t nblocks = (a.ngroups + GPC - 1) / GPC;
  k_translate<D, P, GPC, NT><<<(unsigned)nblocks, NT, smem, Pl->stream>>>(a);
  return cudaGetLastError();
}

#define SFT_DISPATCH(D_, P_, CALL)                     \
  do {                                                 \
    if (D_ == 2 && P_ == 5) { constexpr int D = 2, P = 5; CALL; } \
    else if (D_ == 2 && P_ == 7) { constexpr int D = 2, P = 7; CALL; } \
    else if (D_ == 2 && P_ == 9) { constexpr int D = 2, P = 9; CALL; } \
    else if (D_ == 3 && P_ == 5) { constexpr int D = 3, P = 5; CALL; } \
    else if (D_ == 3 && P_ == 7) { constexpr int D = 3, P = 7; CALL; } \
    else if (D_ == 3 && P_ == 9) { constexpr int D = 3, P = 9; CALL; } \
    else return cudaErrorInvalidValue;                 \
  } while (0)

cudaError_t launch_translate(const sft_plan_s* Pl, const LevelDims& L, const double2* in, double2* out) {
  SFT_DISPATCH(Pl->d, Pl->p, return (launch_translate_t<D, P>(Pl, L, in, out)));
  return cudaSuccess;
}

cudaError_t launch_leaf(const sft_plan_s* Pl, const double2* f, double2* out, int64_t b_lo, int64_t b_hi) {
  if (b_hi <= b_lo) return cudaSuccess;
  const unsigned nb = (unsigned)((b_hi - b_lo + 3) / 4);
  SFT_DISPATCH(Pl->d, Pl->p,
               (k_leaf<D, P><<<nb, 128, 0, Pl->stream>>>(Pl->K.pts_sorted, Pl->K.perm, Pl->K.first_pt, f,
                                                         Pl->tab->leaf_invD, out, b_lo, b_hi, Pl->N)));
  return cudaGetLastError();
}

cudaError_t launch_final(const sft_plan_s* Pl, const double2* g0, double2* u, int64_t a_lo, int64_t a_hi) {
  if (a_hi <= a_lo) return cudaSuccess;
  const unsigned nb = (unsigned)((a_hi - a_lo + 3) / 4);
  SFT_DISPATCH(Pl->d, Pl->p,
               (k_final<D, P><<<nb, 128, 0, Pl->stream>>>(Pl->X.pts_sorted, Pl->X.perm, Pl->X.first_pt, g0, u, a_lo,
                                                          a_hi, Pl->N)));
  return cudaGetLastError();
}

cudaError_t launch_zero(double2* p, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_zero<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(p, n);
  return cudaGetLastError();
}

}  // namespace sft
