/*
 * sft_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for Ying's butterfly sparse
 * Fourier transform (arXiv 0801.1524, /root/reference/PAPER.md = "P:").
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  It shares no code, header,
 * table or helper with the CUDA path (paper_0801_1524_b200/csrc), and the
 * CUDA path never calls it.
 *
 * Precision: long double (x87 80-bit, 64-bit mantissa) for every operation;
 * equivalent charges are stored as double between the two live levels
 * ("only need to keep the equivalent charges for two adjacent
 * levels").  G^{-1} is applied by an LU solve with partial pivoting, never
 * by multiplying with an explicit inverse (reading R1).
 *
 * Functions and the passages they follow:
 *   oracle_direct          eq. (sfft): u_i = sum_j e^{2 pi i x_i.k_j/N} f_j
 *   oracle_G / oracle_H    P:222-224 (G), P:284-286 (H)
 *   oracle_M1 / oracle_E1  eq. (M1) P:213-218 and eq. (E1) P:276-281 as the
 *                          factorised products M11*G*M12 and E11*H*E12
 *   oracle_solve_charges   P:198-212: f = M^{-1} u, M = M1 (x) M2 [(x) M3]
 *   oracle_leaf_charges    §2.2 step 2
 *   oracle_pair_charges    §2.1 fig. 1 + §2.2 step 3
 *   oracle_eval_charges    field of equivalent charges, P:191-197 / step 4 P:306-311
 *   oracle_butterfly       §2.2 steps 1-4
 *   oracle_farfield_direct eq. (far), discretised: u_inf(xhat_i) =
 *                          sum_j e^{-i kappa xhat_i.y_j} F_j (sign s = -1;
 *                          s = +1 gives the adjoint sum)
 *
 * Box conventions (DESIGN.md readings): N = 2^L; level l boxes have width
 * N >> l and integer coordinates c in [0, 2^l)^d, corner c*(N>>l); a point
 * with coordinate y belongs to leaf floor(y) (N-1 when y == N); only
 * non-empty boxes are kept.  Grids include both endpoints,
 * spacing w/(p-1).
 */
#include <complex.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef long double ld;
typedef long double _Complex cld;

static const ld TWO_PI_L = 6.283185307179586476925286766559005768L;

/* e^{2 pi i t} with t reduced to [-1/2, 1/2] first. */
static cld turn(ld t) {
  ld r = t - nearbyintl(t);
  return cosl(TWO_PI_L * r) + I * sinl(TWO_PI_L * r);
}

/* e^{2 pi i num/den} for integers, reduced exactly before the division. */
static cld turn_ratio(int64_t num, int64_t den) {
  int64_t r = num % den;
  if (r < 0) r += den;
  return turn((ld)r / (ld)den);
}

/* ------------------------------------------------------------------ */
/* direct summation, eq. (sfft)                                 */
/* ------------------------------------------------------------------ */
int oracle_direct(int d, double N, const double* x, int64_t nx, const double* k, int64_t nk,
                  const double* f, double* u, const int64_t* targets, int64_t nt, int nthreads) {
  if (d < 1 || d > 3 || N <= 0) return 1;
  int64_t n_out = targets ? nt : nx;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t ii = 0; ii < n_out; ++ii) {
    int64_t i = targets ? targets[ii] : ii;
    cld acc = 0;
    for (int64_t j = 0; j < nk; ++j) {
      ld dot = 0;
      for (int a = 0; a < d; ++a) dot += (ld)x[i * d + a] * (ld)k[j * d + a];
      cld e = turn(dot / (ld)N);
      acc += e * ((ld)f[2 * j] + I * (ld)f[2 * j + 1]);
    }
    u[2 * ii] = (double)creall(acc);
    u[2 * ii + 1] = (double)cimagl(acc);
  }
  return 0;
}

/* Far-field pattern, eq. (far) P:82-96 with the integral replaced by the
 * given quadrature (F_j = f(y_j) ds_j):
 *   u_i = sum_j e^{s i kappa xhat_i . y_j} F_j,  s = -1 (eq. far) or +1 (adjoint).
 * Plain definition in long double, fixed j order; the phase is reduced in
 * turns before the sine/cosine (as in oracle_direct). */
int oracle_farfield_direct(int d, double kappa, int sign, const double* xhat, int64_t nx, const double* y, int64_t ny,
                           const double* F, double* u, int nthreads) {
  if (d < 1 || d > 3 || !(kappa > 0) || (sign != 1 && sign != -1)) return 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t i = 0; i < nx; ++i) {
    cld acc = 0;
    for (int64_t j = 0; j < ny; ++j) {
      ld dot = 0;
      for (int a = 0; a < d; ++a) dot += (ld)xhat[i * d + a] * (ld)y[j * d + a];
      cld e = turn((ld)sign * (ld)kappa * dot / TWO_PI_L);
      acc += e * ((ld)F[2 * j] + I * (ld)F[2 * j + 1]);
    }
    u[2 * i] = (double)creall(acc);
    u[2 * i + 1] = (double)cimagl(acc);
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* fixed matrices G, H and LU of G               */
/* ------------------------------------------------------------------ */
#define PMAX 16

/* (G)_{ll'} = e^{2 pi i l l'/(p-1)^2} */
static cld G_entry(int p, int l, int lp) {
  int64_t P1 = p - 1;
  return turn_ratio((int64_t)l * lp, P1 * P1);
}
/* (H)_{ll'} = e^{pi i l l'/(p-1)^2} = e^{2 pi i l l' / (2 (p-1)^2)} */
static cld H_entry(int p, int l, int lp) {
  int64_t P1 = p - 1;
  return turn_ratio((int64_t)l * lp, 2 * P1 * P1);
}

void oracle_G(int p, double* out) {
  for (int l = 0; l < p; ++l)
    for (int lp = 0; lp < p; ++lp) {
      cld g = G_entry(p, l, lp);
      out[2 * (l * p + lp)] = (double)creall(g);
      out[2 * (l * p + lp) + 1] = (double)cimagl(g);
    }
}
void oracle_H(int p, double* out) {
  for (int l = 0; l < p; ++l)
    for (int lp = 0; lp < p; ++lp) {
      cld h = H_entry(p, l, lp);
      out[2 * (l * p + lp)] = (double)creall(h);
      out[2 * (l * p + lp) + 1] = (double)cimagl(h);
    }
}

typedef struct {
  int p;
  cld lu[PMAX * PMAX];
  int piv[PMAX];
} lu_t;

/* Doolittle LU with partial pivoting of G (long double). */
static void lu_factor_G(int p, lu_t* F) {
  F->p = p;
  for (int l = 0; l < p; ++l)
    for (int m = 0; m < p; ++m) F->lu[l * p + m] = G_entry(p, l, m);
  for (int i = 0; i < p; ++i) F->piv[i] = i;
  for (int c = 0; c < p; ++c) {
    int best = c;
    ld bv = cabsl(F->lu[c * p + c]);
    for (int r = c + 1; r < p; ++r)
      if (cabsl(F->lu[r * p + c]) > bv) { bv = cabsl(F->lu[r * p + c]); best = r; }
    if (best != c) {
      for (int m = 0; m < p; ++m) {
        cld t = F->lu[c * p + m]; F->lu[c * p + m] = F->lu[best * p + m]; F->lu[best * p + m] = t;
      }
      int t = F->piv[c]; F->piv[c] = F->piv[best]; F->piv[best] = t;
    }
    for (int r = c + 1; r < p; ++r) {
      cld fac = F->lu[r * p + c] / F->lu[c * p + c];
      F->lu[r * p + c] = fac;
      for (int m = c + 1; m < p; ++m) F->lu[r * p + m] -= fac * F->lu[c * p + m];
    }
  }
}

/* solve G z = y in place (y -> z) */
static void lu_solve(const lu_t* F, cld* y) {
  int p = F->p;
  cld b[PMAX];
  for (int i = 0; i < p; ++i) b[i] = y[F->piv[i]];
  for (int i = 0; i < p; ++i)
    for (int m = 0; m < i; ++m) b[i] -= F->lu[i * p + m] * b[m];
  for (int i = p - 1; i >= 0; --i) {
    for (int m = i + 1; m < p; ++m) b[i] -= F->lu[i * p + m] * b[m];
    b[i] /= F->lu[i * p + i];
  }
  for (int i = 0; i < p; ++i) y[i] = b[i];
}

/* ------------------------------------------------------------------ */
/* diagonals of eq. (M1) and eq. (E1), one axis                          */
/*   (M1)_{ll'} = e^{2pi i (cA + l wA/P1) cB / N}      -> M11_l            */
/*              * e^{2pi i l l'/P1^2 * wA wB/N}         -> G (wA wB = N)   */
/*              * e^{2pi i cA (l' wB/P1) / N}           -> M12_l'          */
/*   (E1) identical with B -> B_c and wA wBc / N = 1/2 -> H.               */
/* All corners/widths are integers, so each phase is an exact rational   */
/* reduced before conversion to long double.                              */
/* ------------------------------------------------------------------ */
static cld diag_left(int p, int64_t N, int64_t cA, int64_t wA, int64_t cB, int l) {
  int64_t P1 = p - 1;
  return turn_ratio((cA * P1 + (int64_t)l * wA) * cB, P1 * N);
}
static cld diag_right(int p, int64_t N, int64_t cA, int64_t wB, int lp) {
  int64_t P1 = p - 1;
  return turn_ratio(cA * (int64_t)lp * wB, P1 * N);
}

/* M1 = M11 * G * M12 as a dense p x p complex matrix (for pins). */
void oracle_M1(int p, int64_t N, int64_t cA, int64_t wA, int64_t cB, int64_t wB, double* out) {
  for (int l = 0; l < p; ++l)
    for (int lp = 0; lp < p; ++lp) {
      cld v = diag_left(p, N, cA, wA, cB, l) * G_entry(p, l, lp) * diag_right(p, N, cA, wB, lp);
      out[2 * (l * p + lp)] = (double)creall(v);
      out[2 * (l * p + lp) + 1] = (double)cimagl(v);
    }
}
/* E1 = E11 * H * E12 (child box B_c of corner cBc, width wBc). */
void oracle_E1(int p, int64_t N, int64_t cA, int64_t wA, int64_t cBc, int64_t wBc, double* out) {
  for (int l = 0; l < p; ++l)
    for (int lp = 0; lp < p; ++lp) {
      cld v = diag_left(p, N, cA, wA, cBc, l) * H_entry(p, l, lp) * diag_right(p, N, cA, wBc, lp);
      out[2 * (l * p + lp)] = (double)creall(v);
      out[2 * (l * p + lp) + 1] = (double)cimagl(v);
    }
}

/* ------------------------------------------------------------------ */
/* tensor (Kronecker) application along one axis of a p^d array          */
/* ------------------------------------------------------------------ */
static int64_t ipow(int b, int e) {
  int64_t r = 1;
  while (e-- > 0) r *= b;
  return r;
}

typedef struct {
  int d, p, L;
  int64_t N;
  lu_t G;
} ctx_t;

/* y <- E_axis y for E = E11 H E12 on axis a */
static void apply_E_axis(const ctx_t* c, cld* y, int a, int64_t cA, int64_t wA, int64_t cBc, int64_t wBc) {
  int p = c->p, d = c->d;
  int64_t stride = ipow(p, d - 1 - a);
  int64_t total = ipow(p, d);
  cld e11[PMAX], e12[PMAX], H[PMAX * PMAX];
  for (int l = 0; l < p; ++l) {
    e11[l] = diag_left(p, c->N, cA, wA, cBc, l);
    e12[l] = diag_right(p, c->N, cA, wBc, l);
    for (int lp = 0; lp < p; ++lp) H[l * p + lp] = H_entry(p, l, lp);
  }
  for (int64_t base = 0; base < total; ++base) {
    if ((base / stride) % p != 0) continue; /* fiber start: axis-a index 0 */
    cld v[PMAX], w[PMAX];
    for (int l = 0; l < p; ++l) v[l] = e12[l] * y[base + l * stride];
    for (int l = 0; l < p; ++l) {
      cld s = 0;
      for (int lp = 0; lp < p; ++lp) s += H[l * p + lp] * v[lp];
      w[l] = e11[l] * s;
    }
    for (int l = 0; l < p; ++l) y[base + l * stride] = w[l];
  }
}

/* y <- M_axis^{-1} y with M = M11 G M12: conj(M12) G^{-1} conj(M11) */
static void solve_M_axis(const ctx_t* c, cld* y, int a, int64_t cA, int64_t wA, int64_t cB, int64_t wB) {
  int p = c->p, d = c->d;
  int64_t stride = ipow(p, d - 1 - a);
  int64_t total = ipow(p, d);
  cld m11[PMAX], m12[PMAX];
  for (int l = 0; l < p; ++l) {
    m11[l] = diag_left(p, c->N, cA, wA, cB, l);
    m12[l] = diag_right(p, c->N, cA, wB, l);
  }
  for (int64_t base = 0; base < total; ++base) {
    if ((base / stride) % p != 0) continue;
    cld v[PMAX];
    for (int l = 0; l < p; ++l) v[l] = conjl(m11[l]) * y[base + l * stride];
    lu_solve(&c->G, v);
    for (int l = 0; l < p; ++l) y[base + l * stride] = conjl(m12[l]) * v[l];
  }
}

/* f = M^{-1} u on the pair (A,B) given corners/widths per axis. */
static void solve_charges(const ctx_t* c, cld* y, const int64_t* cA, int64_t wA, const int64_t* cB, int64_t wB) {
  for (int a = 0; a < c->d; ++a) solve_M_axis(c, y, a, cA[a], wA, cB[a], wB);
}

static int ctx_init(ctx_t* c, int d, int64_t N, int p) {
  if (d < 2 || d > 3 || p < 3 || p > PMAX || N < 1 || (N & (N - 1))) return 1;
  c->d = d; c->p = p; c->N = N;
  int L = 0;
  while (((int64_t)1 << L) < N) ++L;
  c->L = L;
  lu_factor_G(p, &c->G);
  return 0;
}

/* public: f = M^{-1} u for one pair; u, f are p^d interleaved complex. */
int oracle_solve_charges(int d, int64_t N, int p, const int64_t* cA, int64_t wA, const int64_t* cB, int64_t wB,
                         const double* u, double* f) {
  ctx_t c;
  if (ctx_init(&c, d, N, p)) return 1;
  int64_t n = ipow(p, d);
  cld* y = malloc(sizeof(cld) * n);
  for (int64_t e = 0; e < n; ++e) y[e] = (ld)u[2 * e] + I * (ld)u[2 * e + 1];
  solve_charges(&c, y, cA, wA, cB, wB);
  for (int64_t e = 0; e < n; ++e) { f[2 * e] = (double)creall(y[e]); f[2 * e + 1] = (double)cimagl(y[e]); }
  free(y);
  return 0;
}

/* ------------------------------------------------------------------ */
/* step 2: leaf B of T_K against the root A0 of T_X           */
/* check potentials u_l = sum_{k_j in B} e^{2 pi i x^{A0}_l . k_j / N} f_j, */
/* x^{A0}_l = l N/(p-1) per axis; then f^{A0 B} = M^{-1} u.               */
/* ------------------------------------------------------------------ */
static void leaf_charges(const ctx_t* c, const int64_t* cB, const double* k, const double* f, int64_t n, cld* out) {
  int p = c->p, d = c->d;
  int64_t P1 = p - 1, tot = ipow(p, d);
  for (int64_t e = 0; e < tot; ++e) out[e] = 0;
  for (int64_t j = 0; j < n; ++j) {
    cld fj = (ld)f[2 * j] + I * (ld)f[2 * j + 1];
    /* per axis phase of x^{A0}_l . k_j / N = l * k_j / (p-1): l*k exact in ld,
       fmodl exact, so the phase is exact up to the final division */
    cld ax[3][PMAX];
    for (int a = 0; a < d; ++a)
      for (int l = 0; l < p; ++l) ax[a][l] = turn(fmodl((ld)l * (ld)k[j * d + a], (ld)P1) / (ld)P1);
    for (int64_t e = 0; e < tot; ++e) {
      cld w = fj;
      int64_t r = e;
      for (int a = d - 1; a >= 0; --a) { w *= ax[a][r % p]; r /= p; }
      out[e] += w;
    }
  }
  int64_t cA[3] = {0, 0, 0};
  solve_charges(c, out, cA, c->N, cB, 1);
}

int oracle_leaf_charges(int d, int64_t N, int p, const int64_t* cB, const double* k, const double* f, int64_t n,
                        double* out) {
  ctx_t c;
  if (ctx_init(&c, d, N, p)) return 1;
  int64_t tot = ipow(p, d);
  cld* y = malloc(sizeof(cld) * tot);
  leaf_charges(&c, cB, k, f, n, y);
  for (int64_t e = 0; e < tot; ++e) { out[2 * e] = (double)creall(y[e]); out[2 * e + 1] = (double)cimagl(y[e]); }
  free(y);
  return 0;
}

/* ------------------------------------------------------------------ */
/* step 3 (P:300-305 with fig. 1): one pair (A, B)             */
/* u^{AB} = sum_{present B_c} (E1 (x) E2 [(x) E3]) f^{A' B_c}, then        */
/* f^{AB} = M^{-1} u^{AB}.  A at level L-t (coords ca), B at level t      */
/* (coords cb); child c has bits (axis a <-> bit d-1-a).                  */
/* ------------------------------------------------------------------ */
static void pair_charges(const ctx_t* c, int t, const int64_t* ca, const int64_t* cb, int nchild,
                         const int* child_bits, const double* const* fchild, cld* out) {
  int p = c->p, d = c->d;
  int64_t tot = ipow(p, d);
  int64_t wA = c->N >> (c->L - t), wB = c->N >> t, wBc = c->N >> (t + 1);
  int64_t cA[3], cB[3];
  for (int a = 0; a < d; ++a) { cA[a] = ca[a] * wA; cB[a] = cb[a] * wB; }
  cld* tmp = malloc(sizeof(cld) * tot);
  for (int64_t e = 0; e < tot; ++e) out[e] = 0;
  for (int ch = 0; ch < nchild; ++ch) {
    const double* fc = fchild[ch];
    for (int64_t e = 0; e < tot; ++e) tmp[e] = (ld)fc[2 * e] + I * (ld)fc[2 * e + 1];
    for (int a = 0; a < d; ++a) {
      int bit = (child_bits[ch] >> (d - 1 - a)) & 1;
      int64_t cBc = (2 * cb[a] + bit) * wBc;
      apply_E_axis(c, tmp, a, cA[a], wA, cBc, wBc);
    }
    for (int64_t e = 0; e < tot; ++e) out[e] += tmp[e];
  }
  free(tmp);
  solve_charges(c, out, cA, wA, cB, wB);
}

int oracle_pair_charges(int d, int64_t N, int p, int t, const int64_t* ca, const int64_t* cb, int nchild,
                        const int* child_bits, const double* fchild /* [nchild][p^d] */, double* out) {
  ctx_t c;
  if (ctx_init(&c, d, N, p)) return 1;
  if (t < 0 || t >= c.L || nchild < 0 || nchild > (1 << d)) return 1;
  int64_t tot = ipow(p, d);
  const double* ptrs[8] = {0};
  for (int i = 0; i < nchild; ++i) ptrs[i] = fchild + 2 * tot * i;
  cld* y = malloc(sizeof(cld) * tot);
  pair_charges(&c, t, ca, cb, nchild, child_bits, ptrs, y);
  for (int64_t e = 0; e < tot; ++e) { out[2 * e] = (double)creall(y[e]); out[2 * e + 1] = (double)cimagl(y[e]); }
  free(y);
  return 0;
}

/* ------------------------------------------------------------------ */
/* field of equivalent charges on the grid of box B (corner cB, width wB) */
/* at a point x: sum_l e^{2 pi i x . k^B_l / N} f_l, k^B_l = cB + l wB/P1.  */
/* Used by step 4 with B = B0 (cB = 0, wB = N).               */
/* ------------------------------------------------------------------ */
static cld eval_charges(const ctx_t* c, const int64_t* cB, int64_t wB, const double* f, const double* xpt) {
  int p = c->p, d = c->d;
  int64_t P1 = p - 1, tot = ipow(p, d);
  cld ax[3][PMAX];
  for (int a = 0; a < d; ++a)
    for (int l = 0; l < p; ++l) {
      /* x * (cB + l wB/P1) / N = x (cB P1 + l wB) / (P1 N); the integer factor
         times a double is exact in long double for the sizes used here */
      int64_t q = cB[a] * P1 + (int64_t)l * wB;
      ld ph = fmodl((ld)xpt[a] * (ld)q, (ld)(P1 * c->N)) / (ld)(P1 * c->N);
      ax[a][l] = turn(ph);
    }
  cld acc = 0;
  for (int64_t e = 0; e < tot; ++e) {
    cld w = (ld)f[2 * e] + I * (ld)f[2 * e + 1];
    int64_t r = e;
    for (int a = d - 1; a >= 0; --a) { w *= ax[a][r % p]; r /= p; }
    acc += w;
  }
  return acc;
}

int oracle_eval_charges(int d, int64_t N, int p, const int64_t* cB, int64_t wB, const double* f, const double* x,
                        int64_t nx, double* u) {
  ctx_t c;
  if (ctx_init(&c, d, N, p)) return 1;
  for (int64_t i = 0; i < nx; ++i) {
    cld v = eval_charges(&c, cB, wB, f, x + i * d);
    u[2 * i] = (double)creall(v);
    u[2 * i + 1] = (double)cimagl(v);
  }
  return 0;
}

/* ------------------------------------------------------------------ */
/* step 1: trees of non-empty boxes.  Keys are lexicographic  */
/* (axis 0 most significant): key = sum_a c_a * 2^{l (d-1-a)}.            */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t n;
  int64_t* key; /* sorted unique keys of non-empty boxes at this level */
} level_t;

typedef struct {
  int d, L;
  int64_t npts;
  level_t* lev;      /* [L+1] */
  int64_t* leaf_of;  /* [npts] leaf index of each point */
  int64_t* pt_start; /* [n_leaf+1] CSR of points per leaf */
  int64_t* pt_idx;   /* [npts] */
} tree_t;

static int64_t leaf_coord(double y, int64_t N) {
  int64_t c = (int64_t)floor(y);
  if (c >= N) c = N - 1;
  if (c < 0) c = 0;
  return c;
}

static int64_t make_key(const int64_t* co, int d, int l) {
  int64_t k = 0;
  for (int a = 0; a < d; ++a) k = (k << l) | co[a];
  return k;
}
static void split_key(int64_t key, int d, int l, int64_t* co) {
  int64_t mask = ((int64_t)1 << l) - 1;
  for (int a = d - 1; a >= 0; --a) { co[a] = key & mask; key >>= l; }
}

static int cmp_i64(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

static int64_t find_key(const level_t* lv, int64_t key) {
  int64_t lo = 0, hi = lv->n - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    if (lv->key[mid] == key) return mid;
    if (lv->key[mid] < key) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

static void tree_build(tree_t* T, int d, int L, int64_t N, const double* pts, int64_t n) {
  T->d = d; T->L = L; T->npts = n;
  T->lev = calloc(L + 1, sizeof(level_t));
  int64_t* keys = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  for (int l = L; l >= 0; --l) {
    for (int64_t i = 0; i < n; ++i) {
      int64_t co[3];
      for (int a = 0; a < d; ++a) co[a] = leaf_coord(pts[i * d + a], N) >> (L - l);
      keys[i] = make_key(co, d, l);
    }
    qsort(keys, n, sizeof(int64_t), cmp_i64);
    int64_t m = 0;
    for (int64_t i = 0; i < n; ++i)
      if (i == 0 || keys[i] != keys[i - 1]) keys[m++] = keys[i];
    T->lev[l].n = m;
    T->lev[l].key = malloc(sizeof(int64_t) * (m > 0 ? m : 1));
    memcpy(T->lev[l].key, keys, sizeof(int64_t) * m);
  }
  free(keys);
  int64_t nl = T->lev[L].n;
  T->leaf_of = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  T->pt_start = calloc(nl + 1, sizeof(int64_t));
  T->pt_idx = malloc(sizeof(int64_t) * (n > 0 ? n : 1));
  for (int64_t i = 0; i < n; ++i) {
    int64_t co[3];
    for (int a = 0; a < d; ++a) co[a] = leaf_coord(pts[i * d + a], N);
    T->leaf_of[i] = find_key(&T->lev[L], make_key(co, d, L));
    T->pt_start[T->leaf_of[i] + 1]++;
  }
  for (int64_t b = 0; b < nl; ++b) T->pt_start[b + 1] += T->pt_start[b];
  int64_t* fill = malloc(sizeof(int64_t) * (nl + 1));
  memcpy(fill, T->pt_start, sizeof(int64_t) * (nl + 1));
  for (int64_t i = 0; i < n; ++i) T->pt_idx[fill[T->leaf_of[i]]++] = i; /* ascending i per leaf */
  free(fill);
}

static void tree_free(tree_t* T) {
  for (int l = 0; l <= T->L; ++l) free(T->lev[l].key);
  free(T->lev); free(T->leaf_of); free(T->pt_start); free(T->pt_idx);
}

/* Tree dump for golden tests: per level the count, then keys (lexicographic). */
int oracle_tree_counts(int d, int64_t N, const double* pts, int64_t n, int64_t* counts /* [L+1] */) {
  if (d < 2 || d > 3 || N < 1 || (N & (N - 1))) return 1;
  int L = 0;
  while (((int64_t)1 << L) < N) ++L;
  tree_t T;
  tree_build(&T, d, L, N, pts, n);
  for (int l = 0; l <= L; ++l) counts[l] = T.lev[l].n;
  tree_free(&T);
  return 0;
}

/* ------------------------------------------------------------------ */
/* §2.2 steps 1-4.                                            */
/* Optional restriction for sampled checks at full size: only targets in */
/* `targets` are evaluated (A restricted to their ancestors) and only     */
/* sources with src_active[j] != 0 carry charge (B restricted to boxes    */
/* containing an active source).  Every computed pair uses exactly the    */
/* per-pair arithmetic of the unrestricted run; skipped pairs hold zero   */
/* charges or never reach a sampled target.                              */
/* ------------------------------------------------------------------ */
typedef struct {
  int64_t n;
  int64_t* idx; /* indices into the tree level (ascending) */
} sub_t;

static int64_t sub_find(const sub_t* s, int64_t v) {
  int64_t lo = 0, hi = s->n - 1;
  while (lo <= hi) {
    int64_t mid = (lo + hi) / 2;
    if (s->idx[mid] == v) return mid;
    if (s->idx[mid] < v) lo = mid + 1; else hi = mid - 1;
  }
  return -1;
}

/* mark leaves, then propagate to ancestors: returns per level subsets */
static void ancestors(const tree_t* T, const unsigned char* leaf_mark, sub_t* out /* [L+1] */) {
  int d = T->d, L = T->L;
  unsigned char* mark = malloc(T->lev[L].n > 0 ? T->lev[L].n : 1);
  memcpy(mark, leaf_mark, T->lev[L].n);
  for (int l = L; l >= 0; --l) {
    int64_t cnt = 0;
    for (int64_t b = 0; b < T->lev[l].n; ++b) cnt += mark[b] != 0;
    out[l].n = cnt;
    out[l].idx = malloc(sizeof(int64_t) * (cnt > 0 ? cnt : 1));
    cnt = 0;
    for (int64_t b = 0; b < T->lev[l].n; ++b)
      if (mark[b]) out[l].idx[cnt++] = b;
    if (l == 0) break;
    unsigned char* pm = calloc(T->lev[l - 1].n > 0 ? T->lev[l - 1].n : 1, 1);
    for (int64_t s = 0; s < out[l].n; ++s) {
      int64_t co[3];
      split_key(T->lev[l].key[out[l].idx[s]], d, l, co);
      for (int a = 0; a < d; ++a) co[a] >>= 1;
      pm[find_key(&T->lev[l - 1], make_key(co, d, l - 1))] = 1;
    }
    free(mark);
    mark = pm;
  }
  free(mark);
}

int oracle_butterfly(int d, int64_t N, int p, const double* x, int64_t nx, const double* k, int64_t nk,
                     const double* f, double* u, const int64_t* targets, int64_t nt,
                     const unsigned char* src_active, int nthreads) {
  ctx_t c;
  if (ctx_init(&c, d, N, p)) return 1;
  if (nx < 1 || nk < 1) return 1;
  for (int64_t i = 0; i < nx * d; ++i) if (!(x[i] >= 0 && x[i] <= (double)N)) return 2;
  for (int64_t i = 0; i < nk * d; ++i) if (!(k[i] >= 0 && k[i] <= (double)N)) return 2;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  int L = c.L;
  int64_t tot = ipow(p, d);
  int nchildren = 1 << d;

  /* step 1: trees */
  tree_t TX, TK;
  tree_build(&TX, d, L, N, x, nx);
  tree_build(&TK, d, L, N, k, nk);

  /* restriction sets */
  int64_t n_out = targets ? nt : nx;
  unsigned char* lmX = calloc(TX.lev[L].n, 1);
  for (int64_t ii = 0; ii < n_out; ++ii) lmX[TX.leaf_of[targets ? targets[ii] : ii]] = 1;
  unsigned char* lmK = calloc(TK.lev[L].n, 1);
  for (int64_t j = 0; j < nk; ++j)
    if (!src_active || src_active[j]) lmK[TK.leaf_of[j]] = 1;
  sub_t* SX = calloc(L + 1, sizeof(sub_t));
  sub_t* SK = calloc(L + 1, sizeof(sub_t));
  ancestors(&TX, lmX, SX);
  ancestors(&TK, lmK, SK);
  free(lmX); free(lmK);

  /* step 2: leaf level t = L, pairs (A0, B) for active leaves B */
  double* cur = calloc((size_t)SK[L].n * tot * 2, sizeof(double)); /* [iB][A0] */
  {
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 8)
#endif
    for (int64_t sb = 0; sb < SK[L].n; ++sb) {
      int64_t b = SK[L].idx[sb];
      int64_t co[3];
      split_key(TK.lev[L].key[b], d, L, co);
      int64_t n = TK.pt_start[b + 1] - TK.pt_start[b];
      double* kk = malloc(sizeof(double) * d * (n > 0 ? n : 1));
      double* ff = malloc(sizeof(double) * 2 * (n > 0 ? n : 1));
      int64_t m = 0;
      for (int64_t q = TK.pt_start[b]; q < TK.pt_start[b + 1]; ++q) {
        int64_t j = TK.pt_idx[q];
        if (src_active && !src_active[j]) continue;
        for (int a = 0; a < d; ++a) kk[m * d + a] = k[j * d + a];
        ff[2 * m] = f[2 * j]; ff[2 * m + 1] = f[2 * j + 1];
        ++m;
      }
      cld* y = malloc(sizeof(cld) * tot);
      leaf_charges(&c, co, kk, ff, m, y);
      for (int64_t e = 0; e < tot; ++e) {
        cur[(sb * tot + e) * 2] = (double)creall(y[e]);
        cur[(sb * tot + e) * 2 + 1] = (double)cimagl(y[e]);
      }
      free(y); free(kk); free(ff);
    }
  }

  /* step 3: t = L-1 .. 0; level t holds pairs (A at L-t, B at t), [iB][iA] */
  for (int t = L - 1; t >= 0; --t) {
    const sub_t* SB = &SK[t];
    const sub_t* SA = &SX[L - t];
    const sub_t* SBc = &SK[t + 1];
    const sub_t* SAp = &SX[L - t - 1];
    double* nxt = calloc((size_t)SB->n * SA->n * tot * 2 + 1, sizeof(double));
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t sb = 0; sb < SB->n; ++sb) {
      int64_t cb[3];
      split_key(TK.lev[t].key[SB->idx[sb]], d, t, cb);
      /* present (and active) children B_c */
      int bits[8];
      int64_t cidx[8];
      int nc = 0;
      for (int ch = 0; ch < nchildren; ++ch) {
        int64_t cc[3];
        for (int a = 0; a < d; ++a) cc[a] = 2 * cb[a] + ((ch >> (d - 1 - a)) & 1);
        int64_t bi = find_key(&TK.lev[t + 1], make_key(cc, d, t + 1));
        if (bi < 0) continue;
        int64_t s = sub_find(SBc, bi);
        if (s < 0) continue;
        bits[nc] = ch;
        cidx[nc] = s;
        ++nc;
      }
      cld* y = malloc(sizeof(cld) * tot);
      for (int64_t sa = 0; sa < SA->n; ++sa) {
        int64_t ca[3], cp[3];
        split_key(TX.lev[L - t].key[SA->idx[sa]], d, L - t, ca);
        for (int a = 0; a < d; ++a) cp[a] = ca[a] >> 1;
        int64_t ap = sub_find(SAp, find_key(&TX.lev[L - t - 1], make_key(cp, d, L - t - 1)));
        const double* ptrs[8];
        for (int q = 0; q < nc; ++q) ptrs[q] = cur + ((size_t)cidx[q] * SAp->n + ap) * tot * 2;
        pair_charges(&c, t, ca, cb, nc, bits, ptrs, y);
        double* o = nxt + ((size_t)sb * SA->n + sa) * tot * 2;
        for (int64_t e = 0; e < tot; ++e) { o[2 * e] = (double)creall(y[e]); o[2 * e + 1] = (double)cimagl(y[e]); }
      }
      free(y);
    }
    free(cur);
    cur = nxt; /* only levels t and t+1 were ever live */
  }

  /* step 4: u_i = sum_l e^{2 pi i x_i . k^{B0}_l / N} f^{A B0}_l */
  {
    const sub_t* SA = &SX[L];
    int have_root = SK[0].n > 0;
    int64_t c0[3] = {0, 0, 0};
#ifdef _OPENMP
#pragma omp parallel for schedule(static)
#endif
    for (int64_t ii = 0; ii < n_out; ++ii) {
      int64_t i = targets ? targets[ii] : ii;
      cld v = 0;
      if (have_root) {
        int64_t sa = sub_find(SA, TX.leaf_of[i]);
        v = eval_charges(&c, c0, N, cur + (size_t)sa * tot * 2, x + i * d);
      }
      u[2 * ii] = (double)creall(v);
      u[2 * ii + 1] = (double)cimagl(v);
    }
  }
  free(cur);
  for (int l = 0; l <= L; ++l) { free(SX[l].idx); free(SK[l].idx); }
  free(SX); free(SK);
  tree_free(&TX); tree_free(&TK);
  return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
