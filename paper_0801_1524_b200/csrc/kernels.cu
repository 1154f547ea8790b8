// kernels.cu -- steps 2 and 4 of the butterfly as
// sm_100a FP64 kernels in the box-relative h-representation (sft_internal.cuh,
// DESIGN.md §3).  Step 3 (the per-level translation) is in translate.cu.
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


__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

// ------------------------------------------------------------------------
// K2: leaf kernel, one warp per leaf B of T_K (h-representation)
// ------------------------------------------------------------------------
template <int D, int P, typename T2, int PS>
__global__ __launch_bounds__(128) void k_leaf(const double* __restrict__ k_sorted, const int32_t* __restrict__ perm,
                                              const int32_t* __restrict__ first_pt,
                                              const double2* __restrict__ f, const double* __restrict__ invD,
                                              T2* __restrict__ out, int64_t b_lo, int64_t b_hi, int64_t N) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NACC = (PD + 31) / 32;
  constexpr int P1 = P - 1;
  __shared__ double r_s[4][D][P], sn_s[4][D][P];
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
    // r_m(s) = invD_m prod_{q != m} sin(pi (s P1 - q)/P1^2): lane (a, q) evaluates
    // one sine, lane (a, m) then multiplies the p-1 others
    if (lane < D * P) {
      const int a = lane / P, q = lane % P;
      const double kk = k_sorted[(int64_t)j * D + a];
      const double s = kk - fmin(floor(kk), (double)(N - 1));
      sn_s[warp][a][q] = sinpi((s * P1 - q) / (double)(P1 * P1));
    }
    __syncwarp();
    if (lane < D * P) {
      const int a = lane / P, m = lane % P;
      double prod = invD[m];
#pragma unroll
      for (int q = 0; q < P; ++q)
        if (q != m) prod *= sn_s[warp][a][q];
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
  T2* o = out + (b - b_lo) * (int64_t)PS;
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    const int e = lane + 32 * i;
    if (e < PD) {
      T2 v;
      v.x = acc[i].x;
      v.y = acc[i].y;
      o[e] = v;
    }
  }
}

// ------------------------------------------------------------------------
// K4: final kernel, one warp per leaf A of T_X (h-representation)
// ------------------------------------------------------------------------
template <int D, int P, typename T2, int PS>
__global__ __launch_bounds__(128) void k_final(const double* __restrict__ x_sorted, const int32_t* __restrict__ perm,
                                               const int32_t* __restrict__ first_pt,
                                               const T2* __restrict__ h0, double2* __restrict__ u,
                                               int64_t a_lo, int64_t a_hi, int64_t N) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NACC = (PD + 31) / 32;
  constexpr int P1 = P - 1;
  __shared__ double2 e_s[4][D][P];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t A = a_lo + blockIdx.x * 4 + warp;
  if (A >= a_hi) return;
  const T2* h = h0 + (A - a_lo) * (int64_t)PS;
  double2 hr[NACC];
#pragma unroll
  for (int i = 0; i < NACC; ++i) {
    const int e = lane + 32 * i;
    hr[i] = make_double2(0.0, 0.0);
    if (e < PD) {
      const T2 v = h[e];
      hr[i] = make_double2(v.x, v.y);
    }
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

cudaError_t launch_leaf(const sft_plan_s* Pl, const double2* f, void* out, int64_t b_lo, int64_t b_hi) {
  if (b_hi <= b_lo) return cudaSuccess;
  const unsigned nb = (unsigned)((b_hi - b_lo + 3) / 4);
  if (Pl->prec == 1) {
    SFT_DISPATCH(Pl->d, Pl->p,
                 (k_leaf<D, P, float2, Pow<P, D>::v + (Pow<P, D>::v & 1)><<<nb, 128, 0, Pl->stream>>>(
                     Pl->K.pts_sorted, Pl->K.perm, Pl->K.first_pt, f, Pl->tab->leaf_invD, (float2*)out, b_lo, b_hi,
                     Pl->N)));
  } else {
    SFT_DISPATCH(Pl->d, Pl->p,
                 (k_leaf<D, P, double2, Pow<P, D>::v><<<nb, 128, 0, Pl->stream>>>(
                     Pl->K.pts_sorted, Pl->K.perm, Pl->K.first_pt, f, Pl->tab->leaf_invD, (double2*)out, b_lo, b_hi,
                     Pl->N)));
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_final(const sft_plan_s* Pl, const void* h0, double2* u, int64_t a_lo, int64_t a_hi) {
  if (a_hi <= a_lo) return cudaSuccess;
  const unsigned nb = (unsigned)((a_hi - a_lo + 3) / 4);
  if (Pl->prec == 1) {
    SFT_DISPATCH(Pl->d, Pl->p,
                 (k_final<D, P, float2, Pow<P, D>::v + (Pow<P, D>::v & 1)><<<nb, 128, 0, Pl->stream>>>(
                     Pl->X.pts_sorted, Pl->X.perm, Pl->X.first_pt, (const float2*)h0, u, a_lo, a_hi, Pl->N)));
  } else {
    SFT_DISPATCH(Pl->d, Pl->p,
                 (k_final<D, P, double2, Pow<P, D>::v><<<nb, 128, 0, Pl->stream>>>(
                     Pl->X.pts_sorted, Pl->X.perm, Pl->X.first_pt, (const double2*)h0, u, a_lo, a_hi, Pl->N)));
  }
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
