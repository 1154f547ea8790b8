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
// K2: leaf kernel.  Warp k takes the leaves of T_K whose first source lies in
// the window [W k, W (k+1)) of the sorted sources (W = 24: with <= 8 sources
// per leaf a batch has <= 31 sources; larger leaves are handled in chunks).
// Lane = source: s = k_j - c^B in [0,1]^d, the weights
//   r_m(s_a) = invD_m prod_{q != m} sin(pi (s_a (p-1) - q)/(p-1)^2)
// (one sincospi per axis, sines by angle addition theta - q delta with
// theta = pi s_a/(p-1), delta = pi/(p-1)^2, prefix/suffix products) and the
// rotated charge f_j e^{i pi sum_a s_a}, into shared memory; then, leaf by
// leaf, lane = output element: h^{A0 B}_m = sum_j f'_j prod_a r_{m_a}(s_{j,a}).
// ------------------------------------------------------------------------
// sources per leaf-kernel warp: kLeafWin, or fewer (down to SFT_LEAF_WIN_MIN)
// when the K sources are too few to give every SM four warps at kLeafWin
// (small plans are latency-bound: C1 leaf 13.8 -> 12.3 us at 16 vs 24)
#ifndef SFT_LEAF_WIN
#define SFT_LEAF_WIN 24
#endif
#ifndef SFT_LEAF_WIN_MIN
#define SFT_LEAF_WIN_MIN 12
#endif
constexpr int kLeafWin = SFT_LEAF_WIN;

template <int D, int P>
__device__ __forceinline__ void leaf_weights(const double* __restrict__ k_sorted, int64_t N, int j, const double* cdq,
                                             const double* sdq, const double* inv_s, double (*w)[P], double2* rot,
                                             int ffmod) {
  constexpr int P1 = P - 1;
  double ssum = 0.0;
  int64_t csum = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double kk = k_sorted[(int64_t)j * D + a];
    const double ca = fmin(floor(kk), (double)(N - 1));
    const double sa = kk - ca;  // exact
    ssum += sa;
    csum += (int64_t)ca;
    double sn, cs;
    sincospi(sa / (double)P1, &sn, &cs);
    double sq[P], pre[P];
#pragma unroll
    for (int q = 0; q < P; ++q) sq[q] = fma(sn, cdq[q], -cs * sdq[q]);  // sin(theta - q delta)
    double acc_p = 1.0;
#pragma unroll
    for (int m = 0; m < P; ++m) {
      pre[m] = acc_p;
      acc_p *= sq[m];
    }
    double suf = 1.0;
#pragma unroll
    for (int m = P - 1; m >= 0; --m) {
      w[a][m] = inv_s[m] * pre[m] * suf;
      suf *= sq[m];
    }
  }
  double sn, cs;
  sincospi(ssum, &sn, &cs);
  // far-field adapter (sft_farfield_plan): the charges carry e^{-i pi sum_a k_a}
  // = e^{-i pi sum_a s_a} (-1)^{sum_a c_a}, so the rotation becomes the sign (-1)^{sum c}
  if (ffmod) {
    cs = (csum & 1) ? -1.0 : 1.0;
    sn = 0.0;
  }
  *rot = make_double2(cs, sn);  // e^{i pi sum_a s_a}, applied to each RHS's charge
}

// resident 128-thread blocks per SM the register budget is sized for (leaf / final)
#ifndef SFT_LEAF_MINB2
#define SFT_LEAF_MINB2 6  // C2 leaf 29.5 -> 26 us (4: 120 registers, 20% warps active)
#endif
#ifndef SFT_LEAF_MINB3
#define SFT_LEAF_MINB3 2
#endif
#ifndef SFT_FINAL_MINB2
#define SFT_FINAL_MINB2 1
#endif
#ifndef SFT_FINAL_MINB3
#define SFT_FINAL_MINB3 4  // C3 final 32.8 -> 30.8 us (1, 2: the same 32.8)
#endif
template <int D, int P, typename T2, int PS>
__global__ __launch_bounds__(128, D == 2 ? SFT_LEAF_MINB2 : SFT_LEAF_MINB3) void k_leaf(const double* __restrict__ k_sorted,
                                                              const int32_t* __restrict__ perm,
                                                              const int32_t* __restrict__ first_pt,
                                                              const int32_t* __restrict__ leaf_of,
                                                              const double2* __restrict__ f,
                                                              const double* __restrict__ invD, T2* __restrict__ out,
                                                              int64_t b_lo, int64_t b_hi, int64_t N, int conj,
                                                              int nrhs, int64_t ldf, int64_t ors, int ffmod, int win) {
  constexpr int PD = Pow<P, D>::v;
  constexpr int NACC = (PD + 31) / 32;
  constexpr int P1 = P - 1;
  __shared__ double w_s[4][32][D][P];
  __shared__ double2 f_s[4][32], rot_s[4][32];
  __shared__ double cdq[P], sdq[P], inv_s[P];
  if (threadIdx.x < P) {
    double sn, cs;
    sincospi((double)threadIdx.x / (double)(P1 * P1), &sn, &cs);
    cdq[threadIdx.x] = cs;
    sdq[threadIdx.x] = sn;
    inv_s[threadIdx.x] = invD[threadIdx.x];
  }
  __syncthreads();
  // launched with PDL (launch_pdl): the sources, charges and level buffer are
  // touched only after the previous kernel has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t kw = (int64_t)blockIdx.x * 4 + warp;
  // leaves [lb, le) of this warp: first source in [s0 + W kw, s0 + W (kw+1))
  const int32_t s0 = first_pt[b_lo], s1 = first_pt[b_hi];
  const int64_t w0 = s0 + (int64_t)win * kw, w1 = s0 + (int64_t)win * (kw + 1);
  if (w0 >= s1) return;
  auto lower = [&](int64_t v) {  // first leaf in [b_lo, b_hi] with first_pt >= v (leaf_of: two loads)
    if (v >= s1) return b_hi;
    const int64_t l = leaf_of[v];
    return first_pt[l] >= v ? l : l + 1;
  };
  const int64_t lb = lower(w0), le = lower(w1);
  if (lb >= le) return;
  const int js = first_pt[lb], je = first_pt[le];
  for (int c0 = js; c0 < je; c0 += 32) {
    // weights of the sources [c0, c0 + 32) of this batch
    const int n = min(32, je - c0);
    if (lane < n) leaf_weights<D, P>(k_sorted, N, c0 + lane, cdq, sdq, inv_s, w_s[warp][lane], &rot_s[warp][lane], ffmod);
    const int pj = lane < n ? perm[c0 + lane] : 0;
    // the weights are shared by every RHS of a batch (sft_apply_batch)
    for (int rh = 0; rh < nrhs; ++rh) {
    if (lane < n) {
      double2 fj = f[(int64_t)rh * ldf + pj];
      if (conj) fj.y = -fj.y;
      f_s[warp][lane] = cmul(fj, rot_s[warp][lane]);
    }
    __syncwarp();
    // leaves whose sources intersect [c0, c0 + n)
    for (int64_t b = lb; b < le; ++b) {
      const int jb0 = first_pt[b], jb1 = first_pt[b + 1];
      if (jb1 <= c0 || jb0 >= c0 + n) continue;
      const int t0 = max(jb0, c0) - c0, t1 = min(jb1, c0 + n) - c0;
      T2* o = out + (int64_t)rh * ors + (b - b_lo) * (int64_t)PS;
#pragma unroll
      for (int i = 0; i < NACC; ++i) {
        const int e = lane + 32 * i;
        if (e < PD) {
          double2 acc = make_double2(0.0, 0.0);
          if (jb0 < c0) {  // continuing a leaf from the previous chunk
            const T2 v = o[e];
            acc = make_double2(v.x, v.y);
          }
          for (int t = t0; t < t1; ++t) {
            const double2 fj = f_s[warp][t];
            double w = 1.0;
            int r = e;
#pragma unroll
            for (int a = D - 1; a >= 0; --a) {
              w *= w_s[warp][t][a][r % P];
              r /= P;
            }
            acc.x = fma(w, fj.x, acc.x);
            acc.y = fma(w, fj.y, acc.y);
          }
          T2 v;
          v.x = acc.x;
          v.y = acc.y;
          o[e] = v;
        }
      }
    }
    __syncwarp();
    }
  }
}

// ------------------------------------------------------------------------
// K4: final kernel, one thread per target (32 consecutive sorted targets per
// warp, across leaf boundaries)
// ------------------------------------------------------------------------
// Target x_i in leaf A (xi = x_i - c^A in [0,1]^d): z_a = e^{i pi (2 xi_a - 1)/(p-1)}
// (one sincospi per axis), powers by recurrence, and
//   u_i = sum_l prod_a z_a^{l_a} h^{A B0}_l
// sum-factorised over the axes; h is read through L1 (the ~3 targets of a
// leaf share it).
template <int D, int P, typename T2, int PS>
__global__ __launch_bounds__(128, D == 2 ? SFT_FINAL_MINB2 : SFT_FINAL_MINB3) void k_final(const double* __restrict__ x_sorted, const int32_t* __restrict__ perm,
                                               const int32_t* __restrict__ leaf_of,
                                               const T2* __restrict__ h0, double2* __restrict__ u,
                                               int64_t i_lo, int64_t i_hi, int64_t a_lo, int64_t N, int conj,
                                               int nrhs, int64_t hrs, int64_t ldu, int ffmod) {
  constexpr int P1 = P - 1;
  const int64_t j = i_lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= i_hi) return;
  // launched with PDL (launch_pdl) behind the last translation: the target
  // side (plan data, complete before that translation started) is set up
  // while it drains; h is read after griddepcontrol.wait below
  const int64_t lj = (int64_t)leaf_of[j];
  const T2* const hl = h0 + (lj - a_lo) * (int64_t)PS;
  const int64_t pj = perm ? (int64_t)perm[j] : j - i_lo;  // perm == nullptr: sorted output
  double2 z[D], el[P];
  double xisum = 0.0;
  int64_t csum = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const double xx = x_sorted[j * D + a];
    const double ca = fmin(floor(xx), (double)(N - 1));
    const double xi = xx - ca;  // in [0,1], exact
    xisum += xi;
    csum += (int64_t)ca;
    double sn, cs;
    sincospi((2.0 * xi - 1.0) / (double)P1, &sn, &cs);
    z[a] = make_double2(cs, sn);
  }
  // far-field adapter, adjoint plan: potentials carry e^{i pi sum_a x_a}
  // = (-1)^{sum c} e^{i pi sum xi} (applied after the conjugation)
  double2 fmod_ = make_double2(1.0, 0.0);
  if (ffmod) {
    sincospi(xisum, &fmod_.y, &fmod_.x);
    if (csum & 1) fmod_ = make_double2(-fmod_.x, -fmod_.y);
  }
  el[0] = make_double2(1.0, 0.0);
#pragma unroll
  for (int l = 1; l < P; ++l) el[l] = cmul(el[l - 1], z[D - 1]);
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // the powers are shared by every RHS of a batch (sft_apply_batch)
  for (int rh = 0; rh < nrhs; ++rh) {
  const T2* h = hl + (int64_t)rh * hrs;
  auto inner = [&](int base) {
    double2 t = make_double2(0.0, 0.0);
#pragma unroll
    for (int l = 0; l < P; ++l) {
      const T2 hq = __ldg(h + base + l);
      const double hx = hq.x, hy = hq.y;
      t.x = fma(el[l].x, hx, fma(-el[l].y, hy, t.x));
      t.y = fma(el[l].x, hy, fma(el[l].y, hx, t.y));
    }
    return t;
  };
  double2 s = make_double2(0.0, 0.0);
  double2 w0 = make_double2(1.0, 0.0);
  if constexpr (D == 2) {
#pragma unroll
    for (int l0 = 0; l0 < P; ++l0) {
      const double2 t = inner(l0 * P);
      s.x = fma(w0.x, t.x, fma(-w0.y, t.y, s.x));
      s.y = fma(w0.x, t.y, fma(w0.y, t.x, s.y));
      w0 = cmul(w0, z[0]);
    }
  } else {
#pragma unroll 1
    for (int l0 = 0; l0 < P; ++l0) {
      double2 t1 = make_double2(0.0, 0.0);
      double2 w1 = make_double2(1.0, 0.0);
#pragma unroll
      for (int l1 = 0; l1 < P; ++l1) {
        const double2 t = inner((l0 * P + l1) * P);
        t1.x = fma(w1.x, t.x, fma(-w1.y, t.y, t1.x));
        t1.y = fma(w1.x, t.y, fma(w1.y, t.x, t1.y));
        w1 = cmul(w1, z[1]);
      }
      s.x = fma(w0.x, t1.x, fma(-w0.y, t1.y, s.x));
      s.y = fma(w0.x, t1.y, fma(w0.y, t1.x, s.y));
      w0 = cmul(w0, z[0]);
    }
  }
  if (conj) s.y = -s.y;
  if (ffmod) s = cmul(s, fmod_);
  u[(int64_t)rh * ldu + pj] = s;
  }
}

// Far-field adapter (eq. far): directions xhat (|xhat| = 1) and
// scatterer points y in [0,1]^d become SFT points x = N/2 - kappa xhat/(2 pi),
// k = N y in [0,N]^d, so that 2 pi x.k/N = pi sum_a k_a - kappa xhat.y.
// Rounding can push |x_a - N/2| past N/2 by an ulp when |xhat_a| = 1: such
// points are clamped; anything further out is left for sft_plan's domain check.
__global__ void k_ff_coords(const double* __restrict__ xhat, int64_t nx, const double* __restrict__ y, int64_t ny,
                            int d, double kappa, double N, double* __restrict__ x, double* __restrict__ k) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const double sc = kappa / (2.0 * 3.14159265358979323846);
  if (i < nx * d) {
    double v = 0.5 * N - sc * xhat[i];
    const double tol = 1e-12 * N;
    if (v < 0.0 && v > -tol) v = 0.0;
    if (v > N && v < N + tol) v = N;
    x[i] = v;
  }
  if (i < ny * d) k[i] = N * y[i];
}

cudaError_t launch_ff_coords(const double* xhat, int64_t nx, const double* y, int64_t ny, int d, double kappa,
                             int64_t N, double* x, double* k, cudaStream_t s) {
  const int64_t n = std::max(nx, ny) * d;
  k_ff_coords<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(xhat, nx, y, ny, d, kappa, (double)N, x, k);
  count_launch();
  return cudaGetLastError();
}

__global__ void k_zero(double2* p, int64_t n) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) p[i] = make_double2(0.0, 0.0);
}

// ------------------------------------------------------------------------
// launchers
// ------------------------------------------------------------------------

cudaError_t launch_leaf(const sft_plan_s* Pl, const double2* f, void* out, int64_t b_lo, int64_t b_hi, int nrhs,
                        int64_t ldf, int64_t ors) {
  if (b_hi <= b_lo) return cudaSuccess;
  // sources of leaves [b_lo, b_hi): one warp per window of win sources
  const int64_t ns = b_lo == 0 && b_hi == Pl->K.counts[Pl->L] ? Pl->nk : Pl->k_src_hi - Pl->k_src_lo;
  static PerDevice<int> nsm_;
  int nsm = 0;
  nsm_.get(&nsm, [](int dev, int* r) { return cudaDeviceGetAttribute(r, cudaDevAttrMultiProcessorCount, dev); });
  if (nsm <= 0) nsm = 148;
  const int win = (int)std::max<int64_t>(SFT_LEAF_WIN_MIN, std::min<int64_t>(kLeafWin, ns / (4 * (int64_t)nsm)));
  const int64_t nw = (ns + win - 1) / win;
  const unsigned nb = (unsigned)((nw + 3) / 4);
  if (Pl->prec == 1) {
    SFT_DISPATCH(Pl->d, Pl->p,
                 launch_pdl(k_leaf<D, P, float2, Pow<P, D>::v + (Pow<P, D>::v & 1)>, nb, 128, 0, Pl->stream,
                     Pl->K.pts_sorted, Pl->K.perm, Pl->K.first_pt, Pl->K.leaf_of, f, Pl->tab->leaf_invD, (float2*)out, b_lo, b_hi,
                     Pl->N, Pl->conj, nrhs, ldf, ors, Pl->ffmod && !Pl->conj, win));
  } else {
    SFT_DISPATCH(Pl->d, Pl->p,
                 launch_pdl(k_leaf<D, P, double2, StrideT<double2, Pow<P, D>::v>::v>, nb, 128, 0, Pl->stream,
                     Pl->K.pts_sorted, Pl->K.perm, Pl->K.first_pt, Pl->K.leaf_of, f, Pl->tab->leaf_invD, (double2*)out, b_lo, b_hi,
                     Pl->N, Pl->conj, nrhs, ldf, ors, Pl->ffmod && !Pl->conj, win));
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_final(const sft_plan_s* Pl, const void* h0, double2* u, int64_t a_lo, int64_t i_lo, int64_t i_hi,
                         int nrhs, int64_t hrs, int64_t ldu, bool sorted_out) {
  // targets = sorted points [i_lo, i_hi) of T_X; h0 holds the leaves from a_lo on
  if (i_hi <= i_lo) return cudaSuccess;
  const unsigned nb = (unsigned)((i_hi - i_lo + 127) / 128);
  if (Pl->prec == 1) {
    SFT_DISPATCH(Pl->d, Pl->p,
                 launch_pdl(k_final<D, P, float2, Pow<P, D>::v + (Pow<P, D>::v & 1)>, nb, 128, 0, Pl->stream,
                     Pl->X.pts_sorted, sorted_out ? nullptr : Pl->X.perm, Pl->X.leaf_of, (const float2*)h0, u, i_lo, i_hi, a_lo, Pl->N,
                     Pl->conj, nrhs, hrs, ldu, Pl->ffmod && Pl->conj));
  } else {
    SFT_DISPATCH(Pl->d, Pl->p,
                 launch_pdl(k_final<D, P, double2, StrideT<double2, Pow<P, D>::v>::v>, nb, 128, 0, Pl->stream,
                     Pl->X.pts_sorted, sorted_out ? nullptr : Pl->X.perm, Pl->X.leaf_of, (const double2*)h0, u, i_lo, i_hi, a_lo, Pl->N,
                     Pl->conj, nrhs, hrs, ldu, Pl->ffmod && Pl->conj));
  }
  count_launch();
  return cudaGetLastError();
}

// all-gathered potentials (sorted order, [world][cnt]) to user order
__global__ void k_unsort(const double2* __restrict__ u_all, int64_t cnt, const int64_t* __restrict__ bounds, int world,
                         const int32_t* __restrict__ perm, double2* __restrict__ u, int64_t n) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int q = 0;
  while (q + 1 < world && j >= bounds[q + 1]) ++q;
  u[perm[j]] = u_all[q * cnt + (j - bounds[q])];
}

cudaError_t launch_unsort(const double2* u_all, int64_t cnt, const int64_t* bounds, int world, const int32_t* perm,
                          double2* u, int64_t n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  k_unsort<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(u_all, cnt, bounds, world, perm, u, n);
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
