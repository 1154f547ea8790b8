// tables.cpp -- constant operator tables of the box-relative butterfly,
// built on the host in long double (x87, 64-bit mantissa) and rounded once
// to double.  No explicit G^{-1} is ever formed (reading R1):
// the operators are written with the closed form of the Lagrange basis on
// the nodes z_q = e^{2 pi i q/(p-1)^2} (the columns of G):
//
//   l_m(e^{i phi}) = e^{i P1 (phi - th_m)/2} prod_{q != m} sin((phi - th_q)/2) / sin((th_m - th_q)/2)
//   th_q = 2 pi q / P1^2,  P1 = p - 1.
//
// Translation (P:244-286 with g = M12 f):
//   V[alpha][beta] = e^{i pi alpha beta} W_beta diag(e^{i pi alpha l'/P1}),
//   W_beta[m][l'] = l_m(e^{2 pi i s_l'/P1}),  s_l' = (beta + l'/P1)/2
// i.e. V = M^{-1} E for the child pair expressed in box-relative charges;
// it depends on p only (not on N, level or box position).
// Leaf constants: invD[m] = 1 / prod_{q != m} sin(pi (m - q)/P1^2).
//
// Real form used by the kernels (h-representation, h_m = e^{i pi m/P1} g_m per
// axis): the sine product makes W_beta = diag(e^{-i pi m/P1}) R_beta
// diag(e^{i pi s_l'}) with R_beta REAL, and with D_alpha = C + i s_alpha S
// (C = diag cos(pi l'/(2 P1)), S = diag sin(pi l'/(2 P1)), s_alpha = 2 alpha - 1)
//   T[alpha][beta] = c_{alpha beta} (RC_beta + i s_alpha RS_beta),
//   RC_beta = R_beta C, RS_beta = R_beta S, c = 1 (beta=0), i (alpha=0,beta=1), -i (alpha=1,beta=1),
// so one pair of real p x p products per child gives both alpha outputs.
#include <cmath>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "sft_internal.cuh"

namespace sft {

typedef long double ld;
static const ld PI_L = 3.141592653589793238462643383279502884L;

// l_m(e^{2 pi i s/P1}) for s in [0,1]: returns (re, im) in long double.
static void lagrange_at(int p, int m, ld s, ld* re, ld* im) {
  const int P1 = p - 1;
  ld prod = 1.0L;
  for (int q = 0; q < p; ++q) {
    if (q == m) continue;
    // sin((phi - th_q)/2) = sin(pi (s - q/P1)/P1); sin((th_m - th_q)/2) = sin(pi (m-q)/P1^2)
    ld num = sinl(PI_L * (s * P1 - (ld)q) / ((ld)P1 * P1));
    ld den = sinl(PI_L * (ld)(m - q) / ((ld)P1 * P1));
    prod *= num / den;
  }
  // e^{i P1 (phi - th_m)/2} = e^{i pi (s - m/P1)}
  ld ph = PI_L * (s - (ld)m / P1);
  *re = prod * cosl(ph);
  *im = prod * sinl(ph);
}

void build_tables_host(int p, std::vector<double>& V, std::vector<double>& invD, std::vector<double>* RC,
                       std::vector<double>* RS) {
  const int P1 = p - 1;
  if (RC && RS) {
    RC->assign((size_t)2 * p * p, 0.0);
    RS->assign((size_t)2 * p * p, 0.0);
    for (int be = 0; be < 2; ++be)
      for (int m = 0; m < p; ++m)
        for (int lp = 0; lp < p; ++lp) {
          ld s = ((ld)be + (ld)lp / P1) / 2.0L;
          ld r = 1.0L;
          for (int q = 0; q < p; ++q) {
            if (q == m) continue;
            r *= sinl(PI_L * (s * P1 - (ld)q) / ((ld)P1 * P1)) / sinl(PI_L * (ld)(m - q) / ((ld)P1 * P1));
          }
          ld c = cosl(PI_L * (ld)lp / (2.0L * P1)), sn = sinl(PI_L * (ld)lp / (2.0L * P1));
          (*RC)[((size_t)be * p + m) * p + lp] = (double)(r * c);
          (*RS)[((size_t)be * p + m) * p + lp] = (double)(r * sn);
        }
  }
  V.assign((size_t)2 * 4 * p * p, 0.0);
  for (int al = 0; al < 2; ++al)
    for (int be = 0; be < 2; ++be)
      for (int m = 0; m < p; ++m)
        for (int lp = 0; lp < p; ++lp) {
          ld s = ((ld)be + (ld)lp / P1) / 2.0L;
          ld wr, wi;
          lagrange_at(p, m, s, &wr, &wi);
          // e^{i pi alpha beta} e^{i pi alpha l'/P1}
          ld ph = PI_L * ((ld)(al * be) + (ld)(al * lp) / P1);
          ld cr = cosl(ph), ci = sinl(ph);
          ld vr = wr * cr - wi * ci, vi = wr * ci + wi * cr;
          size_t idx = (((size_t)(al * 2 + be) * p + m) * p + lp);
          V[2 * idx] = (double)vr;
          V[2 * idx + 1] = (double)vi;
        }
  invD.assign(p, 0.0);
  for (int m = 0; m < p; ++m) {
    ld prod = 1.0L;
    for (int q = 0; q < p; ++q)
      if (q != m) prod *= sinl(PI_L * (ld)(m - q) / ((ld)P1 * P1));
    invD[m] = (double)(1.0L / prod);
  }
}

const DeviceTables* get_device_tables(int p, std::string* err) {
  static std::mutex mu;
  static std::map<std::pair<int, int>, DeviceTables*> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    if (err) *err = "cudaGetDevice failed";
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(mu);
  auto key = std::make_pair(dev, p);
  auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  std::vector<double> V, invD, RC, RS;
  build_tables_host(p, V, invD, &RC, &RS);
  DeviceTables* t = new DeviceTables();
  t->p = p;
  if (cudaMalloc(&t->V, V.size() * sizeof(double)) != cudaSuccess ||
      cudaMalloc(&t->leaf_invD, invD.size() * sizeof(double)) != cudaSuccess ||
      cudaMemcpy(t->V, V.data(), V.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(t->leaf_invD, invD.data(), invD.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess) {
    if (err) *err = "table upload failed";
    delete t;
    return nullptr;
  }
  cache[key] = t;
  return t;
}

}  // namespace sft

// Exposed for CPU tests (host only): V [2][2][p][p] complex interleaved, invD [p],
// RC, RS [2][p][p] real (the constant-bank operands of the translation kernel).
extern "C" int sft_operator_tables(int p, double* V, double* invD, double* RC, double* RS) {
  if (p < 3 || p > 15) return SFT_E_ARG;
  std::vector<double> v, d, rc, rs;
  sft::build_tables_host(p, v, d, &rc, &rs);
  if (V)
    for (size_t i = 0; i < v.size(); ++i) V[i] = v[i];
  if (invD)
    for (size_t i = 0; i < d.size(); ++i) invD[i] = d[i];
  if (RC)
    for (size_t i = 0; i < rc.size(); ++i) RC[i] = rc[i];
  if (RS)
    for (size_t i = 0; i < rs.size(); ++i) RS[i] = rs[i];
  return SFT_OK;
}
