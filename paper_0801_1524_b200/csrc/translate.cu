// translate.cu -- step 3 of the butterfly (fig. 1 and eq. E1,
// P:231-286): for every level t = L-1 .. 0 and every group (A', B) with B at
// level t of T_K and A' at level L-t-1 of T_X, the charges of the pairs
// (A, B), A a child of A', from the charges of the pairs (A', B_c):
//
//   h^{AB} = sum_{present B_c} (x)_ax T[alpha_ax][beta_ax] h^{A' B_c},
//   T[a][b] = c_ab (RC_b + i (2a-1) RS_b)   (h-representation)
//
// sum-factorised axis by axis: pass AX combines the two children that differ
// in the bit of axis AX and produces both alpha outputs of that axis at once.
// Per fiber (p complex values along axis AX) and child pair (x_0, x_1):
//
//   z_0 = P - iQ,  z_1 = P + iQ,   P = RC_0 x_0 + RS_1 x_1,  Q = RS_0 x_0 - RC_1 x_1.
//
// Default kernel, k_translate_ws (SFT_TRANSLATE unset or "ws"): a persistent,
// warp-specialised CTA.  The producer warp runs up to NST tiles ahead: for a
// tile of G groups it loads the group metadata, builds per-pass row
// descriptors (one per fiber task: shared-memory position, live children,
// HBM output offsets) and issues 1-D TMA bulk copies of the child arrays into
// a shared-memory stage (mbarrier complete_tx).  NC consumer warps run the
// passes in place in the stage on the FP64 tensor cores: the contraction is a
// real GEMM [fiber rows] x [K = 2p stacked child elements] x [N = (P_m, Q_m)
// interleaved] with mma.sync.m8n8k4.f64 (DMMA -- tcgen05 has no f64 kind);
// the real and imaginary parts of 8 fibers form two A tiles sharing the
// register-resident B fragments, so each lane ends with re and im of (P_m,
// Q_m) and forms z_0, z_1 locally.  K is padded to a multiple of 4 (p=9: 18
// -> 20); the last m of p = 5, 9 runs on DFMA with a 4-lane transpose-reduce
// (N padding avoided: p=9 waste 1.11x instead of 1.78x).  One named barrier
// between passes; the last pass stores straight to HBM.
//
// No floating-point atomics: bitwise reproducible, identical for any world
// size.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <vector>

#include "sft_internal.cuh"

namespace sft {

// ------------------------------------------------------------------------
// shared pieces: arguments, group metadata, TMA tile prologue, task lists
// ------------------------------------------------------------------------
// Per-level layout arguments (everything the schedule builder needs); the
// translation kernels' TransArgs adds the exchange and batch fields.
struct LevelArgs {
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
  // two-level (radix-4) launch, 2D (f2 = 1): levels t+1 and t in one pass over
  // super-groups (A'', B), B at level t of T_K, A'' at level L-t-2 of T_X;
  // cbK/mK: T_K level t, cbK1/mK1: T_K level t+1, cbX/mX: T_X level L-t-1,
  // cbX2/mX2: T_X level L-t-2; input = level t+2 pairs, output = level t
  int f2;
  const int32_t* cbK1;
  const uint32_t* mK1;
  const int32_t* cbX2;
  const uint32_t* mX2;
};

struct TransArgs : LevelArgs {
  // fused exchange (multi-GPU, exchange level): the output pair with send-layout
  // index i in segment q is stored at peer[q] + peer_off[q] + (i - peer_seg[q]) * p^d
  // (the receiving rank's buffer, mapped into this process), i.e. the
  // all-to-all happens in the kernel's epilogue as NVLink peer stores
  int npeer;
  double2* peer[kMaxPeers];
  int64_t peer_off[kMaxPeers];
  int64_t peer_seg[kMaxPeers + 1];
  // multi-RHS batch: work item w = (tile w / nrhs, RHS w % nrhs); RHS r reads
  // in + r * rs and writes out + r * rs (elements of the stored type)
  int nrhs;
  int64_t rs;
  // dynamic tile scheduling: ctr[0] = next work item, ctr[1] = CTAs done
  // fetching (the last one resets both for the next apply); nullptr = static
  // grid-stride assignment
  int* ctr;
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

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

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

// Index of the output pair (child alpha of A', B) in the level output for
// the last pass, -1 if A' has no such child.
__device__ __forceinline__ int64_t out_pair(const LevelArgs& a, const GroupMeta& g, int alpha) {
  if (!(g.mA >> alpha & 1)) return -1;
  const int64_t iA = (int64_t)g.cbX + __popc(g.mA & ((1u << alpha) - 1));
  if (a.nseg == 0) return (g.iB - a.out_b0) * a.out_nA + (iA - a.out_a0);
  int q = 0;
  while (q + 1 < a.nseg && iA >= a.seg[q + 1]) ++q;
  const int64_t wq = a.seg[q + 1] - a.seg[q];
  return a.seg[a.nseg + 1 + q] + (g.iB - a.out_b0) * wq + (iA - a.seg[q]);
}

// ------------------------------------------------------------------------
// DMMA kernel
// ------------------------------------------------------------------------
// Child-grid structure: a child box has half the width and the
// same p nodes, so its even nodes l' = 2i coincide with parent nodes
// (s (p-1) = (beta (p-1) + l')/2 is an integer) and the Lagrange basis is a
// delta there: column l' of RC_beta / RS_beta is zero except at row
// m = (beta (p-1) + l')/2.  Only the H = (p-1)/2 odd columns per child are
// dense.
//
// Mirror symmetry: the child-1 grid is the mirror image of the child-0 grid
// about the parent's centre (node l' of child 1 sits at 1 - node (p-1-l') of
// child 0, parent node m at 1 - node p-1-m), and the Lagrange basis on the
// nodes z_m = e^{2 pi i m/(p-1)^2} maps to its conjugate under the mirror, so
//   RC_1 = J RS_0 J,  RS_1 = J RC_0 J         (J = index reversal)
// (checked on the host tables to the last bit; tests/test_library_host.py).
// With y = J x_1, s = x_0 + y, t = x_0 - y and m' = p-1-m, the pass
//   P = RC_0 x_0 + RS_1 x_1,  Q = RS_0 x_0 - RC_1 x_1
// becomes, for m < H,
//   P_m = SP_m + DP_m,  P_m' = SP_m - DP_m,  Q_m = SQ_m + DQ_m,  Q_m' = SQ_m - DQ_m,
//   SP_m = 1/2 (RC_0[m] + RC_0[m']) . s,   DP_m = 1/2 (RC_0[m] - RC_0[m']) . t,
//   SQ_m = 1/2 (RS_0[m] + RS_0[m']) . t,   DQ_m = 1/2 (RS_0[m] - RS_0[m']) . s,
// and at the centre P_H = RC_0[H] . s, Q_H = RS_0[H] . t: half the MACs of
// the direct form.  On the tensor cores (DMMA m8n8k4, row = fiber, real and
// imaginary parts of 8 fibers as two A tiles sharing the B fragments) the odd
// elements of s and of t are one k-step each (K = H <= 4); the s-GEMM's
// columns are (SP_m, DQ_m) interleaved and the t-GEMM's (DP_m, SQ_m), so lane
// c of a row holds m = c and forms z_0 = P - iQ, z_1 = P + iQ for m and m'
// locally.  The centre sits in the same N tile for p = 5, 7 (lane c = H:
// columns (SP_H, 0) and (0, SQ_H), so the m and m' formulas coincide) and for
// p = 9 is a DFMA tail (4-lane transpose-reduce).  The even (delta) elements
// start the accumulators: lane c takes s and t at element 2c.
// p = 9: the centre column m = H as a DFMA tail with a 4-lane transpose-reduce
// (0, default) or on a second DMMA N tile (1: 144 fewer static instructions
// but +4 DMMA per super-tile; measured C2 translate 0.997 vs 0.979 ms -- the
// FP64 pipe, which DMMA and DFMA share, is the busier resource)
#ifndef SFT_CENTRE_DMMA
#define SFT_CENTRE_DMMA 0
#endif
template <int P>
struct SymShape {
  static constexpr int H = (P - 1) / 2;   // odd (dense) elements per child = k of the MMA (padded to 4)
  static constexpr bool TAIL = H >= 4;    // centre column outside the 8-column tile (p = 9)
  static_assert(H <= 4, "p <= 9");
  // fragment table (doubles, 32 lanes each): B_s, B_t, delta (s-acc col 0/1, t-acc col 0/1),
  // tail (s coefficient, t coefficient, s delta, t delta; p = 9)
  static constexpr int OFF_BS = 0, OFF_BT = 32, OFF_DS = 64, OFF_DT = 128, OFF_TAIL = 192;
  static constexpr int NFRAG = OFF_TAIL + (TAIL ? 4 * 32 : 0);
};

// p = 5 keeps the direct (child-stacked) form: K = 4 = the two odd elements of
// each child in one k-step, N = (P_m, Q_m) for m = 0..3 in one tile, m = 4 a
// DFMA tail -- 2 DMMA per super-tile; the symmetric form would need 4 (its
// s- and t-GEMMs each fill only half a k-step) plus the sum/difference adds.
#ifndef SFT_SYM5
#define SFT_SYM5 0
#endif
template <int P>
struct UseSym {
  static constexpr bool v = P >= 7 || (SFT_SYM5 && P == 5);
};
#ifndef SFT_CLASS_SPLIT
// class-uniform super-tiles skip the absent child's loads; 2D symmetric form
// only (measured: C2 translate 0.948 -> 0.942 ms; 3D: C3 0.750 -> 0.833, C4
// 33.8 -> 35.5 ms -- three instantiations of the 3D passes cost more)
#define SFT_CLASS_SPLIT 1
#endif
#ifndef SFT_CLASS_SPLIT3
#define SFT_CLASS_SPLIT3 0  // 3D too
#endif
#ifndef SFT_SLOTPAD
#define SFT_SLOTPAD 0  // 1: measured no gain (C3 0.758 vs 0.756 ms)
#endif
// Stage: child slot c of group j at c * SLOT + j * PS elements, SLOT = G * PS +
// SlotPad.  The direct form reads both children in one instruction (lanes 0, 1:
// child 0; lanes 2, 3: child 1), so their slots must not be a multiple of 8
// 16-byte units apart (G * p^d is, e.g. 3D p = 5 with G = 2 on axis 0: 1000):
// one element of padding per child slot makes the step odd.  The symmetric
// form loads the two children in separate instructions: no padding.
// (in elements of the array stride PS: FP64 p^d is odd; the FP32 stride is even
// and a pad would break the 16-byte alignment of the bulk copies, so none)
template <int D, int P, int PS>
struct SlotPad {
  static constexpr int v = (!UseSym<P>::v && (PS & 1)) ? SFT_SLOTPAD : 0;
};
struct DirShape5 {
  static constexpr int P = 5;
  // fragment table: B, tail (P, Q weights of this lane's k), delta (a0, b0, a1, b1) of m = lane%4, tail delta
  static constexpr int OFF_B = 0, OFF_TAIL = 32, OFF_DELTA = 96, OFF_DTAIL = 224, NFRAG = 288;
};

// complex element of the level buffers / stages: double2 (FP64) or float2
// (FP32 storage variant; the arithmetic stays FP64 on the tensor cores)
template <typename E>
struct ElemT;
template <>
struct ElemT<double2> {
  using scalar = double;
  __device__ __forceinline__ static double2 ld(const double2& v) { return v; }
  __device__ __forceinline__ static double2 mk(double re, double im) { return make_double2(re, im); }
};
template <>
struct ElemT<float2> {
  using scalar = float;
  __device__ __forceinline__ static double2 ld(const float2& v) { return make_double2(v.x, v.y); }
  __device__ __forceinline__ static float2 mk(double re, double im) { return make_float2((float)re, (float)im); }
};
// pair-array stride (elements) in buffers and stages: FP32 arrays padded to an
// even count so every array is a multiple of 16 bytes (bulk copies)

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// Stage accesses by 32-bit shared-memory address (explicit ld/st.shared: the
// row bases are selected between a stage slot and the zero slot, which
// generic pointers would turn into generic LD/ST).  volatile: never moved
// across the pass barriers and stage waits (also volatile asm).
template <typename E>
__device__ __forceinline__ double2 lds(uint32_t a);
// How the consumers see absent children (a task's class bit clear):
// 2 = the row reads the CTA's zero slot (default); 0 = the producer zero-fills
// their slots (measured on one box: C2 0.975 vs 0.989 ms, C4 36.5 vs 36.8 ms)
#ifndef SFT_ABSENT
#define SFT_ABSENT 2
#endif
template <>
__device__ __forceinline__ double2 lds<double2>(uint32_t a) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(a));
  return v;
}
template <>
__device__ __forceinline__ double2 lds<float2>(uint32_t a) {
  float x, y;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(x), "=f"(y) : "r"(a));
  return make_double2(x, y);
}
template <typename E>
__device__ __forceinline__ void sts(uint32_t a, double re, double im) {
  if constexpr (sizeof(E) == 16)
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(re), "d"(im) : "memory");
  else
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"((float)re), "f"((float)im) : "memory");
}
template <typename E>
__device__ __forceinline__ void sts1(uint32_t a, double v) {
  if constexpr (sizeof(E) == 16)
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
  else
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"((float)v) : "memory");
}

// One output array of a row: in place in the stage (shared address s) or, in
// the last pass, in HBM / a peer's buffer (GL, pointer g); ok = false: no store.
template <typename E, bool GL>
struct OutRow {
  E* g;
  uint32_t s;
  bool ok;
  __device__ __forceinline__ void st(int el, double re, double im) const {
    if (!ok) return;
#if defined(SFT_ABL_NOGSTORE) || defined(SFT_ABL_NOSSTORE)  // ablation: values kept live, not stored
#ifdef SFT_ABL_NOGSTORE
    if constexpr (GL) { asm volatile("" ::"d"(re), "d"(im)); return; }
#endif
#ifdef SFT_ABL_NOSSTORE
    if constexpr (!GL) { asm volatile("" ::"d"(re), "d"(im)); return; }
#endif
#endif
    if constexpr (GL) g[el] = ElemT<E>::mk(re, im);
    else sts<E>(s + el * (int)sizeof(E), re, im);
  }
  __device__ __forceinline__ void st1(int el, int comp, double v) const {  // real (0) or imaginary (1) part
    if (!ok) return;
    if constexpr (GL) reinterpret_cast<typename ElemT<E>::scalar*>(g + el)[comp] = (typename ElemT<E>::scalar)v;
    else sts1<E>(s + el * (int)sizeof(E) + comp * (int)sizeof(typename ElemT<E>::scalar), v);
  }
};

// Per-lane operator registers of the symmetric pass (lane c = lane % 4)
template <int P>
struct LaneOps {
  using S = SymShape<P>;
  double bs, bt;            // B fragments: s- and t-GEMM, k = c, column lane / 4
                            // (direct form, p = 5: bs = B, bt unused)
  double ds0, ds1, dt0, dt1;  // delta coefficients of this lane's accumulator columns (even element 2c)
                              // (direct form: a0, b0, a1, b1 of m = c)
  double ts, tt, tds, tdt;    // p = 9 centre: odd coefficients of this lane's k, centre deltas (lane 0)
                              // (direct form: tail P / Q weights of this lane's k, tail delta on lane 0)
  double b2;                  // direct form, SFT_TAIL5_DMMA: B fragment of the tail tile (columns P_4, Q_4)
};

template <int P>
__device__ __forceinline__ void load_lane_ops(LaneOps<P>& op, const double* __restrict__ frag, int lane) {
  if constexpr (!UseSym<P>::v) {
    using S = DirShape5;
    op.bs = frag[S::OFF_B + lane];
    op.bt = 0.0;
    op.ts = frag[S::OFF_TAIL + lane];
    op.tt = frag[S::OFF_TAIL + 32 + lane];
    op.ds0 = frag[S::OFF_DELTA + lane];
    op.ds1 = frag[S::OFF_DELTA + 32 + lane];
    op.dt0 = frag[S::OFF_DELTA + 64 + lane];
    op.dt1 = frag[S::OFF_DELTA + 96 + lane];
    op.tds = frag[S::OFF_DTAIL + lane];
    op.tdt = frag[S::OFF_DTAIL + 32 + lane];
    op.b2 = (lane >> 2) == 0 ? op.ts : (lane >> 2) == 1 ? op.tt : 0.0;  // B[k = lane % 4][n = lane / 4]
    return;
  }
  using S = SymShape<P>;
  op.bs = frag[S::OFF_BS + lane];
  op.bt = frag[S::OFF_BT + lane];
  op.ds0 = frag[S::OFF_DS + lane];
  op.ds1 = frag[S::OFF_DS + 32 + lane];
  op.dt0 = frag[S::OFF_DT + lane];
  op.dt1 = frag[S::OFF_DT + 32 + lane];
  if constexpr (S::TAIL) {
    op.ts = frag[S::OFF_TAIL + lane];
    op.tt = frag[S::OFF_TAIL + 32 + lane];
    op.tds = frag[S::OFF_TAIL + 64 + lane];
    op.tdt = frag[S::OFF_TAIL + 96 + lane];
  } else {
    op.ts = op.tt = op.tds = op.tdt = 0.0;
  }
  op.b2 = 0.0;
}

// ------------------------------------------------------------------------
// Tile schedule (built once per plan by k_schedule, read by the producer)
// ------------------------------------------------------------------------
// Per tile of G consecutive groups (B-major, A' fastest) one block of BLK
// bytes in HBM:
//   cnt[NCNT][3] int32: per list (3D: per round and axis), task counts of class both / bit-0 only / bit-1 only
//   grp[G]     {pin0, mB}: pair index of the first child array (iB_c, iA') in the
//              level input, and the child mask of B (children r at pin0 + r*in_nA)
//   task[D][MAXT] TaskRec, per pass packed in class order
// A task = (group j, beta-prefix, alpha-suffix) of pass AX: the fibers of the
// stage slots (bp,0,as) / (bp,1,as).
struct __align__(16) TaskRec {
  uint32_t x;    // stage offset (complex) of the slot with axis bit 0: (j*2^d + slot0)*p^d
  uint32_t cls;  // bit 0 / bit 1: the slot with axis bit 0 / 1 holds data
  uint32_t o0;   // last pass: output offset (complex) from a.out of child alpha-bit 0 of A'; ~0u = absent
  uint32_t o1;   //            ... alpha-bit 1
};

template <int D, int P, int G>
struct Sched {
  static constexpr int MAXT = G << (D - 1);  // tasks per pass (max)
  // task lists: 2D: list 1 = first pass on axis 1 and list 0 = last pass on
  // axis 0 (default order); list 2 = first pass on axis 0 and list 3 = last
  // pass on axis 1 (groups whose reversed axis order needs fewer tasks).
  // 3D: list r = round r of the three passes; every group runs its own axis
  // order (schedule_round3), so list r holds three sub-lists, one per axis
  // (2, 1, 0 in that order), each class-sorted, with count triplets
  // cnt[3 r + k] for the sub-list of axis 2 - k.
  static constexpr int NL = D == 2 ? 4 : D;
  static constexpr int NCNT = D == 2 ? 4 : 9;             // count triplets
  static constexpr int HDR = (NCNT * 12 + 15) / 16 * 16;  // int cnt[NCNT][3]
  static constexpr int GRP = (8 * G + 15) / 16 * 16;
  static constexpr int BLK = HDR + GRP + NL * MAXT * (int)sizeof(TaskRec);
  __device__ __forceinline__ static const int* cnt(const unsigned char* b) { return reinterpret_cast<const int*>(b); }
  __device__ __forceinline__ static const uint2* grp(const unsigned char* b) {
    return reinterpret_cast<const uint2*>(b + HDR);
  }
  __device__ __forceinline__ static const TaskRec* task(const unsigned char* b, int ax) {
    return reinterpret_cast<const TaskRec*>(b + HDR + GRP) + ax * MAXT;
  }
};

// Task lists of pass AX for one tile: the tile's G groups sit in G adjacent
// lanes (a warp holds 32/G tiles); entries packed in class order with scans
// over the G-lane segment.
// REV (2D only): the axes are processed in the order 0, 1 instead of 1, 0.
// Pass over axis 0 first: tasks by beta_1 (slots (0,b1), (1,b1)); then axis 1
// (last): tasks by alpha_0 (slots (a0,0), (a0,1)), outputs (a0,0), (a0,1).
// Stage layout: slot-major, child slot c of group j at stage slot c * G + j
// (the G groups' arrays of one child slot are contiguous: one bulk copy when
// the tile's groups share B and have consecutive A').  TR (two-level launch,
// second level, G = 4k virtual groups): group alpha of super-group sg reads
// child c at stage slot alpha * G + 4 sg + c -- the first level left pair
// (A'_alpha, B_c) in slot alpha of virtual group 4 sg + c -- so its slot pairs
// are 1 slot apart instead of G
template <int D, int P, int G, int PS, int AX, bool LAST, bool REV = false, bool TR = false>
__device__ __forceinline__ void schedule_pass(const LevelArgs& a, const GroupMeta& m, bool valid, bool write_cnt,
                                              int* cnt, TaskRec* out) {
  constexpr int PD = PS;  // offsets in units of the array stride
  constexpr int NS = 1 << D;
  constexpr int SH = D - 1 - AX;
  constexpr int NE = 1 << (D - 1);
  static_assert(!REV || D == 2, "reversed axis order is 2D only");
  const int lane = threadIdx.x & 31;
  TaskRec mine[NE];
  int n = 0, c3 = 0, c1 = 0, c2 = 0;
  if (REV && valid) {
    // AX == 0 first: task b1 in {b1 : some (b0,b1) present}, slots (0,b1)/(1,b1)
    // AX == 1 last:  task a0 in proj_hi(mA,1), slots (a0,0)/(a0,1), class = beta_1 presence
    const uint32_t b1set = proj_lo<D>(m.mB, 1), a0set = proj_hi<D>(m.mA, 1);
#pragma unroll
    for (int v = 0; v < 2; ++v) {
      if (!((AX == 0 ? b1set : a0set) >> v & 1)) continue;
      TaskRec t;
      uint32_t cls;
      int slot0;
      if (AX == 0) {
        cls = (m.mB >> v & 1u) | ((m.mB >> (2 + v) & 1u) << 1);  // (0,b1), (1,b1)
        slot0 = v;
      } else {
        cls = b1set;
        slot0 = v << 1;
      }
      t.x = TR ? (uint32_t)(((lane % NS) * G + ((lane % G) & ~(NS - 1)) + slot0) * PD)
               : (uint32_t)(slot0 * (G * PD + SlotPad<D, P, PD>::v) + (lane % G) * PD);
      t.cls = cls;
      t.o0 = t.o1 = ~0u;
      if (LAST) {
        const int64_t q0 = out_pair(a, m, v << 1), q1 = out_pair(a, m, (v << 1) | 1);
        if (q0 >= 0) t.o0 = (uint32_t)(q0 * PD);
        if (q1 >= 0) t.o1 = (uint32_t)(q1 * PD);
      }
      mine[n++ & (NE - 1)] = t;
      c3 += cls == 3;
      c1 += cls == 1;
      c2 += cls == 2;
    }
  }
  if (!REV && valid) {
    const uint32_t PBp = AX > 0 ? proj_hi<D>(m.mB, AX) : 1u;
    const uint32_t PAs = proj_lo<D>(m.mA, D - 1 - AX);
    const uint32_t PBa = proj_hi<D>(m.mB, AX + 1);
#pragma unroll
    for (int bp = 0; bp < (1 << AX); ++bp) {
      if (!(PBp >> bp & 1)) continue;
      const uint32_t cls = (PBa >> (bp << 1)) & 3u;
#pragma unroll
      for (int as = 0; as < (1 << (D - 1 - AX)); ++as) {
        if (!(PAs >> as & 1)) continue;
        TaskRec t;
        const int sl = (bp << (D - AX)) | as;
        t.x = TR ? (uint32_t)(((lane % NS) * G + ((lane % G) & ~(NS - 1)) + sl) * PD)
                 : (uint32_t)(sl * (G * PD + SlotPad<D, P, PD>::v) + (lane % G) * PD);
        t.cls = cls;
        t.o0 = t.o1 = ~0u;
        if (LAST) {
          const int64_t q0 = out_pair(a, m, as), q1 = out_pair(a, m, (1 << SH) | as);
          if (q0 >= 0) t.o0 = (uint32_t)(q0 * PD);
          if (q1 >= 0) t.o1 = (uint32_t)(q1 * PD);
        }
        mine[n++ & (NE - 1)] = t;
        c3 += cls == 3;
        c1 += cls == 1;
        c2 += cls == 2;
      }
    }
  }
  const int j = lane % G;
  int o3 = c3, o1 = c1, o2 = c2;
#pragma unroll
  for (int d = 1; d < G; d <<= 1) {
    const int t3 = __shfl_up_sync(0xffffffffu, o3, d, G), t1 = __shfl_up_sync(0xffffffffu, o1, d, G),
              t2 = __shfl_up_sync(0xffffffffu, o2, d, G);
    if (j >= d) {
      o3 += t3;
      o1 += t1;
      o2 += t2;
    }
  }
  const int n3 = __shfl_sync(0xffffffffu, o3, G - 1, G), n1 = __shfl_sync(0xffffffffu, o1, G - 1, G);
  const int n2 = __shfl_sync(0xffffffffu, o2, G - 1, G);
  o3 -= c3;
  o1 += n3 - c1;
  o2 += n3 + n1 - c2;
#pragma unroll
  for (int q = 0; q < NE; ++q) {
    if (q < n) {
      const TaskRec t = mine[q];
      out[t.cls == 3 ? o3++ : (t.cls == 1 ? o1++ : o2++)] = t;
    }
  }
  if (j == 0 && write_cnt) {
    cnt[0] = n3;
    cnt[1] = n1;
    cnt[2] = n2;
  }
}

// ---- 3D: per-group axis order --------------------------------------------
#ifndef SFT_ORDER3
#define SFT_ORDER3 1
#endif
#ifndef SFT_ROUND_UNROLL
#define SFT_ROUND_UNROLL 1  // 3D rounds 0, 1 unrolled (C3 translate 0.737 -> 0.715 ms, C4 32.8 -> 32.2)
#endif
// Projection of a child mask onto a set of axes: bit (c & sel) set for every
// present child c, sel = the slot bits (bit D-1-a for axis a) of the axes kept.
__device__ __forceinline__ uint32_t proj_sel(uint32_t m, uint32_t sel) {
  uint32_t r = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c)
    if (m >> c & 1) r |= 1u << (c & sel);
  return r;
}
__device__ __forceinline__ uint32_t axbit3(int a) { return 1u << (2 - a); }

// Fiber tasks of a group under axis order (o1, o2, o3): pass on o1: one per
// present beta over {o2, o3}; on o2: per present alpha_o1 x beta_o3; on o3: per
// present alpha over {o1, o2}.
__device__ __forceinline__ int order_tasks3(uint32_t mB, uint32_t mA, int o1, int o2, int o3) {
  const uint32_t b1 = axbit3(o1), b2 = axbit3(o2), b3 = axbit3(o3);
  return __popc(proj_sel(mB, b2 | b3)) + __popc(proj_sel(mA, b1)) * __popc(proj_sel(mB, b3)) +
         __popc(proj_sel(mA, b1 | b2));
}

// The axis order of a 3D group with the fewest fiber tasks, from its own
// masks only (identical for any partition of the work); ties keep the
// earlier order of the list, whose first entry (2, 1, 0) is the default.
// Returns o1 | o2 << 2 | o3 << 4.  (The tasks are 16% fewer than with the
// fixed order on C3 and 18% on C4; the translation time is linear in them.)
__device__ __forceinline__ uint32_t best_order3(uint32_t mB, uint32_t mA) {
  constexpr uint32_t ords[6] = {2u | 1u << 2 | 0u << 4, 2u | 0u << 2 | 1u << 4, 1u | 2u << 2 | 0u << 4,
                                1u | 0u << 2 | 2u << 4, 0u | 2u << 2 | 1u << 4, 0u | 1u << 2 | 2u << 4};
  uint32_t best = ords[0];
  int bt = order_tasks3(mB, mA, 2, 1, 0);
#pragma unroll
  for (int i = 1; i < 6; ++i) {
    const int t = order_tasks3(mB, mA, ords[i] & 3, ords[i] >> 2 & 3, ords[i] >> 4 & 3);
    if (t < bt) {
      bt = t;
      best = ords[i];
    }
  }
  return best;
}

// Round R (0, 1, 2) of a 3D group's passes under its order ord: the pass on
// axis ax = o_{R+1}, alpha over the axes done before (Aset), beta over the
// axes still to come (Bset).  Task = (alpha over Aset, beta over Bset): the
// fibers of slots (.., beta_ax = 0, ..) / (.., 1, ..); class bit v = the slot
// with beta_ax = v holds data, i.e. (v, beta over Bset) is a projection of a
// present child of B onto {ax} u Bset.  Writes the round's three sub-lists
// (axis 2, 1, 0), class-sorted, with scans over the G-lane segment.
template <int D, int P, int G, int PS, int R>
__device__ __forceinline__ void schedule_round3(const LevelArgs& a, const GroupMeta& m, uint32_t ord, bool valid,
                                                bool write_cnt, int* cnt, TaskRec* out) {
  static_assert(D == 3, "3D rounds");
  constexpr int PD = PS;
  constexpr bool LAST = R == 2;
  const int lane = threadIdx.x & 31;
  const int ax = (int)(ord >> (2 * R) & 3u);
  uint32_t selA = 0, selB = 0;
#pragma unroll
  for (int q = 0; q < 3; ++q) {
    const uint32_t b = axbit3((int)(ord >> (2 * q) & 3u));
    if (q < R) selA |= b;
    if (q > R) selB |= b;
  }
  const uint32_t bax = axbit3(ax);
  const uint32_t pA = proj_sel(m.mA, selA), pB = proj_sel(m.mB, selB), pBa = proj_sel(m.mB, selB | bax);
  TaskRec mine[4];
  int n = 0;
  int cc[3] = {0, 0, 0};  // class 3 / 1 / 2 counts
  if (valid) {
    // alpha and beta bits live in disjoint slot bits: enumerate sl over the
    // subsets of selA | selB
    const uint32_t selAB = selA | selB;
    for (uint32_t sl = 0; sl < 8u; ++sl) {
      if (sl & ~selAB) continue;
      if (!(pA >> (sl & selA) & 1u) || !(pB >> (sl & selB) & 1u)) continue;
      const uint32_t sb = sl & selB;
      const uint32_t cls = (pBa >> sb & 1u) | ((pBa >> (sb | bax) & 1u) << 1);
      TaskRec t;
      t.x = (uint32_t)(sl * (G * PD + SlotPad<D, P, PD>::v) + (lane % G) * PD);
      t.cls = cls;
      t.o0 = t.o1 = ~0u;
      if (LAST) {
        const int64_t q0 = out_pair(a, m, (int)sl), q1 = out_pair(a, m, (int)(sl | bax));
        if (q0 >= 0) t.o0 = (uint32_t)(q0 * PD);
        if (q1 >= 0) t.o1 = (uint32_t)(q1 * PD);
      }
      mine[n++ & 3] = t;
      cc[cls == 3 ? 0 : (cls == 1 ? 1 : 2)]++;
    }
  }
  // per (sub-list k = 2 - ax, class) exclusive offsets over the segment
  const int k = 2 - ax;
  int v[9], tot[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) v[i] = (valid && i / 3 == k) ? cc[i % 3] : 0;
  const int j = lane % G;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    int s = v[i];
#pragma unroll
    for (int d = 1; d < G; d <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, s, d, G);
      if (j >= d) s += t;
    }
    tot[i] = __shfl_sync(0xffffffffu, s, G - 1, G);
    v[i] = s - v[i];  // exclusive
  }
  int base = 0, off[3] = {0, 0, 0};
#pragma unroll
  for (int kk = 0; kk < 3; ++kk) {
    if (kk == k) {
      off[0] = base + v[3 * kk];
      off[1] = base + tot[3 * kk] + v[3 * kk + 1];
      off[2] = base + tot[3 * kk] + tot[3 * kk + 1] + v[3 * kk + 2];
    }
    base += tot[3 * kk] + tot[3 * kk + 1] + tot[3 * kk + 2];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (q < n) {
      const TaskRec t = mine[q];
      out[t.cls == 3 ? off[0]++ : (t.cls == 1 ? off[1]++ : off[2]++)] = t;
    }
  }
  if (j == 0 && write_cnt) {
#pragma unroll
    for (int i = 0; i < 9; ++i) cnt[i] = tot[i];
  }
}

// 2D axis order per group (from its own masks only, so identical for any
// partition of the work and for single- or two-level launches): the order
// with fewer fiber tasks over its two passes -- axis 1 first: one task per
// present beta_0, then one per present alpha_1; axis 0 first: per present
// beta_1, then per present alpha_0.  true = axis 0 first.
template <int P>
__device__ __forceinline__ bool reversed_order(const GroupMeta& m) {
#ifdef SFT_FIXED_ORDER
  return false;
#else
  constexpr int D = 2;
  const int cf = __popc(proj_hi<D>(m.mB, 1)) + __popc(proj_lo<D>(m.mA, 1));
  const int cr = __popc(proj_lo<D>(m.mB, 1)) + __popc(proj_hi<D>(m.mA, 1));
  return cr < cf;
#endif
}

// Two-level tile (2D, f2): lane j of the G-lane segment is virtual group
// v = j (super-group sg = j / 4 of the tile, child c = j % 4).  Two schedule
// blocks per tile, each in the single-level format (lists 1/2 first passes,
// 0/3 second passes, per-group axis order as in single-level launches, so
// the arithmetic and the bits are the same):
//   block 0, first level (levels t+2 -> t+1): group (A'', B_c), its children
//     B_cc at level t+2 in slots v*4 + c', both passes in place, leaving pair
//     (A'_alpha, B_c) in slot v*4 + alpha; block 0 also holds the group
//     records the producer loads from;
//   block 1, second level (t+1 -> t): group (A'_alpha, B), alpha = j % 4,
//     reading its children on the transposed slots sg*16 + c*4 + alpha (TR),
//     the second pass to HBM.
// Absent B_c leave zero-filled slots (they contribute nothing); absent A'_alpha
// have no second-level group.
template <int D, int P, int G, int PS>
__device__ __forceinline__ void schedule_f2(const LevelArgs& a, int64_t tile, bool tv, unsigned char* b) {
  using SC = Sched<D, P, G>;
  constexpr int NS = 1 << D;
  const int lane = threadIdx.x & 31;
  const int j = lane % G;
  const int64_t sgi = tile * (G / NS) + j / NS;  // super-group index
  const int cj = j % NS;
  const bool sv = tv && sgi * NS < a.ngroups;
  GroupMeta m1, m2;
  m1.iB = m1.iAp = m2.iB = m2.iAp = 0;
  m1.cbK = m1.cbX = m2.cbK = m2.cbX = 0;
  m1.mB = m1.mA = m2.mB = m2.mA = 0;
  bool v1 = false, v2 = false;
  if (sv) {
    const uint32_t nap = (uint32_t)a.nAp_grp;
    const int64_t iB = a.b_lo + sgi / nap, iA2 = a.ap_lo + sgi % nap;
    const uint32_t mBB = a.mK[iB], mA2 = a.mX2[iA2];
    const int32_t cbB = a.cbK[iB], cbA2 = a.cbX2[iA2];
    // first level: (A'', B_c), c = cj
    v1 = (mBB >> cj) & 1u;
    if (v1) {
      const int64_t iBc = cbB + __popc(mBB & ((1u << cj) - 1u));
      m1.iB = iBc;
      m1.iAp = iA2;
      m1.cbK = a.cbK1[iBc];
      m1.mB = a.mK1[iBc];
      m1.cbX = cbA2;
      m1.mA = mA2;
    }
    // second level: (A'_alpha, B), alpha = cj
    v2 = (mA2 >> cj) & 1u;
    if (v2) {
      const int64_t iAp = cbA2 + __popc(mA2 & ((1u << cj) - 1u));
      m2.iB = iB;
      m2.iAp = iAp;
      m2.cbK = cbB;
      m2.mB = mBB;
      m2.cbX = a.cbX[iAp];
      m2.mA = a.mX[iAp];
    }
  }
  unsigned char* b1 = b + SC::BLK;
  if (tv) {
    const int64_t pin0 = ((int64_t)m1.cbK - a.in_b0) * a.in_nA + (m1.iAp - a.in_a0);
    reinterpret_cast<uint2*>(b + SC::HDR)[j] = v1 ? make_uint2((uint32_t)pin0, m1.mB) : make_uint2(0u, 0u);
    reinterpret_cast<uint2*>(b1 + SC::HDR)[j] = make_uint2(0u, 0u);
  }
  const bool r1 = v1 && reversed_order<P>(m1), r2 = v2 && reversed_order<P>(m2);
  int* c0 = reinterpret_cast<int*>(b);
  TaskRec* k0 = reinterpret_cast<TaskRec*>(b + SC::HDR + SC::GRP);
  schedule_pass<D, P, G, PS, 1, false>(a, m1, v1 && !r1, tv, c0 + 3, k0 + SC::MAXT);
  schedule_pass<D, P, G, PS, 0, false>(a, m1, v1 && !r1, tv, c0, k0);
  schedule_pass<D, P, G, PS, 0, false, true>(a, m1, v1 && r1, tv, c0 + 6, k0 + 2 * SC::MAXT);
  schedule_pass<D, P, G, PS, 1, false, true>(a, m1, v1 && r1, tv, c0 + 9, k0 + 3 * SC::MAXT);
  int* c1 = reinterpret_cast<int*>(b1);
  TaskRec* k1 = reinterpret_cast<TaskRec*>(b1 + SC::HDR + SC::GRP);
  schedule_pass<D, P, G, PS, 1, false, false, true>(a, m2, v2 && !r2, tv, c1 + 3, k1 + SC::MAXT);
  schedule_pass<D, P, G, PS, 0, true, false, true>(a, m2, v2 && !r2, tv, c1, k1);
  schedule_pass<D, P, G, PS, 0, false, true, true>(a, m2, v2 && r2, tv, c1 + 6, k1 + 2 * SC::MAXT);
  schedule_pass<D, P, G, PS, 1, true, true, true>(a, m2, v2 && r2, tv, c1 + 9, k1 + 3 * SC::MAXT);
}

// All levels of a plan in one launch: level lv owns the global tiles
// [tile0[lv], tile0[lv+1]) and writes its blocks at dst[lv].
constexpr int kSchedChunk = 16;  // levels per schedule launch (the struct is one < 4 KB kernel parameter)
struct SchedLevels {
  LevelArgs a[kSchedChunk];
  unsigned char* dst[kSchedChunk];
  int* ctr[kSchedChunk];  // the launch's tile counters, zeroed here (nullptr: none)
  int64_t tile0[kSchedChunk + 1];
  int nlev;
};
static_assert(sizeof(SchedLevels) <= 4096, "k_schedule's parameter must stay within 4 KB");

// F2K: the two-level (f2) levels' schedules (a separate instantiation, so the
// single-level builder keeps its registers and occupancy)
template <int D, int P, int G, int PS, bool F2K = false>
__global__ __launch_bounds__(128) void k_schedule(const __grid_constant__ SchedLevels S) {
  using SC = Sched<D, P, G>;
  static_assert(G >= 1 && G <= 32 && (G & (G - 1)) == 0, "G must be a power of two");
  constexpr int TPW = 32 / G;  // tiles per warp (G-lane segments)
  const int lane = threadIdx.x & 31;
  if (blockIdx.x == 0 && threadIdx.x < 2 * S.nlev && S.ctr[threadIdx.x >> 1]) S.ctr[threadIdx.x >> 1][threadIdx.x & 1] = 0;
  const int64_t T = ((int64_t)blockIdx.x * 4 + (threadIdx.x >> 5)) * TPW + lane / G;  // global tile
  const int j = lane % G;
  if (T - lane / G >= S.tile0[S.nlev]) return;  // whole warp out of range
  int lv = 0;
  while (lv + 1 < S.nlev && T >= S.tile0[lv + 1]) ++lv;
  const LevelArgs& a = S.a[lv];
  const int64_t tile = T - S.tile0[lv];
  const bool tv = T < S.tile0[S.nlev];
  if constexpr (F2K) {
    if constexpr (D == 2 && G % 4 == 0) schedule_f2<D, P, G, PS>(a, tile, tv, S.dst[lv] + (tv ? tile : 0) * (2 * SC::BLK));
    return;
  }
  unsigned char* b = S.dst[lv] + (tv ? tile : 0) * SC::BLK;
  const int64_t g = tile * G + j;
  const bool valid = tv && g < a.ngroups;
  GroupMeta m;
  m.iB = m.iAp = 0;
  m.cbK = m.cbX = 0;
  m.mB = m.mA = 0;
  if (valid) {
    const uint32_t gg = (uint32_t)g, nap = (uint32_t)a.nAp_grp;
    const uint32_t q = gg / nap;
    m.iB = a.b_lo + q;
    m.iAp = a.ap_lo + (gg - q * nap);
    m.cbK = a.cbK[m.iB];
    m.mB = a.mK[m.iB];
    m.cbX = a.cbX[m.iAp];
    m.mA = a.mX[m.iAp];
  }
  if (tv) {
    const int64_t pin0 = ((int64_t)m.cbK - a.in_b0) * a.in_nA + (m.iAp - a.in_a0);
    reinterpret_cast<uint2*>(b + SC::HDR)[j] = valid ? make_uint2((uint32_t)pin0, m.mB) : make_uint2(0u, 0u);
  }
  int* cnt = reinterpret_cast<int*>(b);  // written by the first lane of each valid tile only
  TaskRec* tk = reinterpret_cast<TaskRec*>(b + SC::HDR + SC::GRP);
  if constexpr (D == 2) {
    const bool rev = valid && reversed_order<P>(m);
    schedule_pass<D, P, G, PS, 1, false>(a, m, valid && !rev, tv, cnt + 3, tk + SC::MAXT);
    schedule_pass<D, P, G, PS, 0, true>(a, m, valid && !rev, tv, cnt, tk);
    schedule_pass<D, P, G, PS, 0, false, true>(a, m, valid && rev, tv, cnt + 6, tk + 2 * SC::MAXT);
    schedule_pass<D, P, G, PS, 1, true, true>(a, m, valid && rev, tv, cnt + 9, tk + 3 * SC::MAXT);
  } else {
    // per-group axis order (SFT_ORDER3=0: the fixed order 2, 1, 0)
    const uint32_t ord = (SFT_ORDER3 && valid) ? best_order3(m.mB, m.mA) : (2u | 1u << 2);
    schedule_round3<D, P, G, PS, 0>(a, m, ord, valid, tv, cnt, tk);
    schedule_round3<D, P, G, PS, 1>(a, m, ord, valid, tv, cnt + 9, tk + SC::MAXT);
    schedule_round3<D, P, G, PS, 2>(a, m, ord, valid, tv, cnt + 18, tk + 2 * SC::MAXT);
  }
}

// Schedule invariants (debug: SFT_CHECK_SCHED=1 at plan time): one thread
// per tile checks counts, stage offsets, classes and HBM offsets against the
// level sizes; any violation sets *err (bit 2).
template <int D, int P, int G>
__global__ void k_check_schedule(TransArgs a, const unsigned char* __restrict__ sched, int64_t ntiles,
                                 int64_t in_pairs, int64_t out_pairs, int* err) {
  using SC = Sched<D, P, G>;
  constexpr int PD = StrideT<double2, Pow<P, D>::v>::v;  // offsets are in units of the array stride
  constexpr int STAGE = (1 << D) * (G * PD + SlotPad<D, P, PD>::v);
  const int64_t tile = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (tile >= ntiles) return;
  const unsigned char* b = sched + tile * SC::BLK;
  bool bad = false;
  for (int j = 0; j < G; ++j) {
    const uint2 gr = SC::grp(b)[j];
    const int np = __popc(gr.y);
    if (np > 0 && (int64_t)gr.x + (int64_t)(np - 1) * a.in_nA >= in_pairs) bad = true;
  }
  // lists: 2D one count triplet each; 3D three (sub-lists of axes 2, 1, 0)
  constexpr int SUB = D == 2 ? 1 : 3;
  for (int l = 0; l < SC::NL; ++l) {
    const int* c = SC::cnt(b) + 3 * SUB * l;
    int nt = 0;
    for (int q = 0; q < 3 * SUB; ++q) {
      if (c[q] < 0) bad = true;
      nt += c[q];
    }
    if (nt > SC::MAXT) bad = true;
    const bool last = D == 2 ? (l == 0 || l == 3) : l == 2;
    for (int t = 0; t < nt && t < SC::MAXT; ++t) {
      const TaskRec r = SC::task(b, l)[t];
      if (r.x >= STAGE || r.cls < 1 || r.cls > 3) bad = true;
      if (last) {
        if (r.o0 != ~0u && (int64_t)r.o0 / PD >= out_pairs) bad = true;
        if (r.o1 != ~0u && (int64_t)r.o1 / PD >= out_pairs) bad = true;
      }
    }
  }
  if (bad) atomicOr(err, 4);
}

#ifndef SFT_ROTATE
#define SFT_ROTATE 1
#endif
#ifndef SFT_ROTATE3
#define SFT_ROTATE3 1  // 3D too: C4 translate 34.4 -> 33.5 ms, C3 0.789 -> 0.783 ms
#endif
// NSUB super-tiles per warp iteration (independent MMA chains interleaved),
// per (d, p); SFT_NSUB overrides all
#ifdef SFT_NSUB
#define SFT_NSUB25 SFT_NSUB
#define SFT_NSUB27 SFT_NSUB
#define SFT_NSUB29 SFT_NSUB
#define SFT_NSUB35 SFT_NSUB
#define SFT_NSUB37 SFT_NSUB
#endif
#ifndef SFT_NSUB25
#define SFT_NSUB25 1
#endif
#ifndef SFT_NSUB27
#define SFT_NSUB27 1
#endif
#ifndef SFT_NSUB29
#define SFT_NSUB29 1
#endif
#ifndef SFT_NSUB35
#define SFT_NSUB35 1
#endif
#ifndef SFT_NSUB37
#define SFT_NSUB37 1
#endif
template <int D, int P>
struct NsubCfg {
  static constexpr int v = D == 2 ? (P == 5 ? SFT_NSUB25 : P == 7 ? SFT_NSUB27 : SFT_NSUB29)
                                  : (P == 5 ? SFT_NSUB35 : P == 7 ? SFT_NSUB37 : 1);
};
// SFT_TAIL5_DMMA=1: the direct form's tail m = p-1 on a second DMMA N tile
// (columns P_4, Q_4 on lane c = 0 of each row) instead of per-lane partials
// and a 4-lane transpose-reduce (6 SHFL, selects and adds per super-tile)
#ifndef SFT_TAIL5_DMMA
#define SFT_TAIL5_DMMA 1  // C3 translate 0.713 -> 0.684 ms, C2 geometry at p = 5 0.423 -> 0.399; 89 -> 80 registers
#endif
// Row -> fiber map of a super-tile (shared-memory bank conflicts, and whole
// sectors for the HBM stores of a last pass).  The symmetric form uses the
// identity with the store-order swap of consumer_pass (scripts/rfib_model_sym.py).
template <int D, int P, int AX, bool LAST>
struct RowMap {
  __device__ __forceinline__ static int fiber(int r) {
    // symmetric form, and any pass storing to HBM: consecutive fibers in rows
    // 2q, 2q+1 (a store instruction then fills whole 32-byte sectors)
    if constexpr (UseSym<P>::v || LAST) return r;
    // direct form (p = 5), in-place passes: scripts/rfib_search_direct.py (slot-major stage, G of WsCfg)
    else if constexpr (D == 2) return (0x43726150u >> (4 * r)) & 7;                     // 0 5 1 6 2 7 3 4
    else if constexpr (AX == 1 || (AX == 0 && SFT_TAIL5_DMMA))
      return (0x76432150u >> (4 * r)) & 7;  // 0 5 1 2 3 4 6 7 (axis 0: with the merged tail-delta load, G = 1)
    else return (0x73625140u >> (4 * r)) & 7;                                           // 0 4 1 5 2 6 3 7
  }
};

// Super-tile arithmetic of the direct form (p = 5, DirShape5): lane c loads
// child (c >> 1)'s odd element 2 (c & 1) + 1 (the A fragment of k = c), and
// for its output m = c child 0's element 2m and child 1's element 2m - (p-1)
// (the delta columns, coefficients 0 when out of range); 2 DMMA give (P_m,
// Q_m) of m = c, a 4-lane transpose-reduce the tail m = p-1.
template <int D, int P, int STR, int C1, int NSUB, typename E, bool GL, int PRES>
__device__ __forceinline__ void direct_math(const LaneOps<P>& op, const uint32_t (&xa)[NSUB], const uint32_t (&xb)[NSUB],
                                            const OutRow<E, GL> (&o0)[NSUB], const OutRow<E, GL> (&o1)[NSUB], int c) {
  constexpr int ES = sizeof(E);
  const int o_a = (2 * (c & 1) + 1) * STR * ES;  // of child c >> 1 (byte offsets)
  // (DMMA tail: lanes c = 0, 1 have no child-1 delta column, so lane 0's
  // child-1 load fetches the tail delta, element p-1, instead -- one load less)
  const int o_e0 = min(2 * c, P - 1) * STR * ES,
            o_e1 = (SFT_TAIL5_DMMA && c == 0 ? P - 1 : max(2 * c - (P - 1), 0)) * STR * ES;
  const int o_t = (P - 1) * STR * ES;  // tail delta: child 1, element p-1
  double are[NSUB][2], aim[NSUB][2], tl[NSUB][4];
  double avx[NSUB], avy[NSUB];
#pragma unroll
  for (int u = 0; u < NSUB; ++u) {
    // PRES (warp-uniform): 1 = no row of the super-tile has child 1, 2 = none
    // has child 0 -- that child's loads are skipped (zeros); 3 = rows may
    // lack either (an absent child reads the zero slot)
    const double2 z = make_double2(0.0, 0.0);
    const double2 av = (c >> 1) ? (PRES & 2 ? lds<E>(xb[u] + o_a) : z) : (PRES & 1 ? lds<E>(xa[u] + o_a) : z);
    const double2 x0 = PRES & 1 ? lds<E>(xa[u] + o_e0) : z;
    const double2 x1 = PRES & 2 ? lds<E>(xb[u] + o_e1) : z;
    const double2 xt = SFT_TAIL5_DMMA ? x1 : (PRES & 2 ? lds<E>(xb[u] + o_t) : z);
    are[u][0] = fma(op.dt0, x1.x, op.ds0 * x0.x);
    are[u][1] = fma(op.dt1, x1.x, op.ds1 * x0.x);
    aim[u][0] = fma(op.dt0, x1.y, op.ds0 * x0.y);
    aim[u][1] = fma(op.dt1, x1.y, op.ds1 * x0.y);
    if constexpr (SFT_TAIL5_DMMA) {
      // tail tile accumulators: (P_4, Q_4) deltas on lane c = 0 (tds, tdt are 0 elsewhere)
      tl[u][0] = op.tds * xt.x;
      tl[u][1] = op.tdt * xt.x;
      tl[u][2] = op.tds * xt.y;
      tl[u][3] = op.tdt * xt.y;
    } else {
      tl[u][0] = fma(av.x, op.ts, op.tds * xt.x);  // P.re
      tl[u][1] = fma(av.x, op.tt, op.tdt * xt.x);  // Q.re
      tl[u][2] = fma(av.y, op.ts, op.tds * xt.y);  // P.im
      tl[u][3] = fma(av.y, op.tt, op.tdt * xt.y);  // Q.im
    }
    avx[u] = av.x;
    avy[u] = av.y;
  }
#ifndef SFT_ABL_NOCOMPUTE
#pragma unroll
  for (int u = 0; u < NSUB; ++u) {
    dmma(are[u], avx[u], op.bs);
    dmma(aim[u], avy[u], op.bs);
    if constexpr (SFT_TAIL5_DMMA) {
      double (&tr)[2] = *reinterpret_cast<double(*)[2]>(&tl[u][0]);
      double (&ti)[2] = *reinterpret_cast<double(*)[2]>(&tl[u][2]);
      dmma(tr, avx[u], op.b2);
      dmma(ti, avy[u], op.b2);
    }
  }
#endif
  const bool odd = c & 1, hi = c & 2;
#pragma unroll
  for (int u = 0; u < NSUB; ++u) {
    o0[u].st(c * STR, are[u][0] + aim[u][1], aim[u][0] - are[u][1]);  // z_0 = P - iQ
    o1[u].st(c * STR, are[u][0] - aim[u][1], aim[u][0] + are[u][1]);  // z_1 = P + iQ
    if constexpr (SFT_TAIL5_DMMA) {
      // lane c = 0: tl = (P_4.re, Q_4.re, P_4.im, Q_4.im)
      if (c == 0) {
        o0[u].st((P - 1) * STR, tl[u][0] + tl[u][3], tl[u][2] - tl[u][1]);
        o1[u].st((P - 1) * STR, tl[u][0] - tl[u][3], tl[u][2] + tl[u][1]);
      }
      continue;
    }
    // tail m = p-1: (z_0.re, z_0.im, z_1.re, z_1.im) partials, transpose-reduce
    const double u0 = tl[u][0] + tl[u][3], u1 = tl[u][2] - tl[u][1];
    const double u2 = tl[u][0] - tl[u][3], u3 = tl[u][2] + tl[u][1];
    double va = odd ? u1 : u0, vb = odd ? u3 : u2;
    va += __shfl_xor_sync(0xffffffffu, odd ? u0 : u1, 1);
    vb += __shfl_xor_sync(0xffffffffu, odd ? u2 : u3, 1);
    double w = hi ? vb : va;
    w += __shfl_xor_sync(0xffffffffu, hi ? va : vb, 2);
    (hi ? o1[u] : o0[u]).st1((P - 1) * STR, c & 1, w);
  }
}

// Which row of a 16-byte phase swaps the m / m' store order (see consumer_pass):
// the even rows where the odd-row swap would put both rows' first stores on the
// same bank groups (scripts/rfib_model_sym.py: 3D p = 7 axes 1, 2 and 2D p = 7)
template <int D, int P, int AX>
struct SwapEven {
  static constexpr bool v = P == 7 && (D == 2 || AX >= 1);
};

// Super-tile arithmetic of the symmetric form (p = 7, 9; see SymShape)
template <int D, int P, int STR, int C1, int NSUB, typename E, bool GL, int PRES>
__device__ __forceinline__ void sym_math(const LaneOps<P>& op, const uint32_t (&xa)[NSUB], const uint32_t (&xb)[NSUB],
                                         const OutRow<E, GL> (&o0)[NSUB], const OutRow<E, GL> (&o1)[NSUB],
                                         int c, int o_a0, int o_a1, int o_d0, int o_d1, int o_f, int o_s, bool st_f,
                                         bool st_s, double sg) {
  using S = SymShape<P>;
  using ET = ElemT<E>;
  constexpr int H = S::H;
  // accumulators: s-GEMM columns (SP_m, DQ_m), t-GEMM columns (DP_m, SQ_m), re / im rows
  double sre[NSUB][2], sim[NSUB][2], tre[NSUB][2], tim[NSUB][2], tl[NSUB][4];
  double ar[NSUB][2], ai[NSUB][2];  // odd s / t of this lane's k (re, im)
  double csr[NSUB][2], csi[NSUB][2], ctr[NSUB][2], cti[NSUB][2], cre[NSUB][2], cim[NSUB][2];  // centre tile (p = 9)
#pragma unroll
  for (int u = 0; u < NSUB; ++u) {
    constexpr int ES = sizeof(E);
    // PRES (warp-uniform, see direct_math): s = x0 + Jx1, t = x0 - Jx1 with the
    // absent child's loads skipped (s = t = x0, or s = -t = Jx1)
    double2 e0 = make_double2(0.0, 0.0), e1 = e0, a0 = e0, a1 = e0;
    if constexpr (PRES & 1) {
      e0 = lds<E>(xa[u] + o_d0 * ES);
      a0 = lds<E>(xa[u] + o_a0 * ES);
    }
    if constexpr (PRES & 2) {
      e1 = lds<E>(xb[u] + o_d1 * ES);
      a1 = lds<E>(xb[u] + o_a1 * ES);
    }
    double ser, sei, ter, tei;
    if constexpr (PRES == 3) {
      ser = e0.x + e1.x; sei = e0.y + e1.y; ter = e0.x - e1.x; tei = e0.y - e1.y;
    } else if constexpr (PRES == 1) {
      ser = ter = e0.x; sei = tei = e0.y;
    } else {
      ser = e1.x; sei = e1.y; ter = -e1.x; tei = -e1.y;
    }
    sre[u][0] = op.ds0 * ser;
    sre[u][1] = op.ds1 * ser;
    sim[u][0] = op.ds0 * sei;
    sim[u][1] = op.ds1 * sei;
    tre[u][0] = op.dt0 * ter;
    tre[u][1] = op.dt1 * ter;
    tim[u][0] = op.dt0 * tei;
    tim[u][1] = op.dt1 * tei;
    if constexpr (PRES == 3) {
      ar[u][0] = a0.x + a1.x;  // s
      ai[u][0] = a0.y + a1.y;
      ar[u][1] = a0.x - a1.x;  // t
      ai[u][1] = a0.y - a1.y;
    } else if constexpr (PRES == 1) {
      ar[u][0] = ar[u][1] = a0.x;
      ai[u][0] = ai[u][1] = a0.y;
    } else {
      ar[u][0] = a1.x;
      ai[u][0] = a1.y;
      ar[u][1] = -a1.x;
      ai[u][1] = -a1.y;
    }
    if constexpr (S::TAIL && SFT_CENTRE_DMMA) {
      // centre m = H (p = 9) on a second N tile: column 0 = SP_H (s-GEMM) and
      // SQ_H (t-GEMM), both on lane c = 0 of the row; centre delta (s, t at
      // element p-1) starts the accumulators there
      const double2 c0 = PRES & 1 ? lds<E>(xa[u] + (P - 1) * STR * ES) : make_double2(0.0, 0.0);
      const double2 c1 = PRES & 2 ? lds<E>(xb[u]) : make_double2(0.0, 0.0);
      cre[u][0] = op.tds * (c0.x + c1.x);
      cim[u][0] = op.tds * (c0.y + c1.y);
      cre[u][1] = op.tdt * (c0.x - c1.x);
      cim[u][1] = op.tdt * (c0.y - c1.y);
      csr[u][1] = csi[u][1] = ctr[u][1] = cti[u][1] = 0.0;
      csr[u][0] = cre[u][0];
      csi[u][0] = cim[u][0];
      ctr[u][0] = cre[u][1];
      cti[u][0] = cim[u][1];
    } else if constexpr (S::TAIL) {
      // centre m = H (p = 9): partials of z_0, z_1 over this lane's k, centre delta on lane 0
      const double2 c0 = PRES & 1 ? lds<E>(xa[u] + (P - 1) * STR * ES) : make_double2(0.0, 0.0);
      const double2 c1 = PRES & 2 ? lds<E>(xb[u]) : make_double2(0.0, 0.0);
      const double pr = fma(op.tds, c0.x + c1.x, op.ts * ar[u][0]), pi = fma(op.tds, c0.y + c1.y, op.ts * ai[u][0]);
      const double qr = fma(op.tdt, c0.x - c1.x, op.tt * ar[u][1]), qi = fma(op.tdt, c0.y - c1.y, op.tt * ai[u][1]);
      tl[u][0] = pr + qi;
      tl[u][1] = pi - qr;
      tl[u][2] = pr - qi;
      tl[u][3] = pi + qr;
    }
  }
#ifndef SFT_ABL_NOCOMPUTE  // ablation: no tensor-core work
#pragma unroll
  for (int u = 0; u < NSUB; ++u) {
    dmma(sre[u], ar[u][0], op.bs);
    dmma(sim[u], ai[u][0], op.bs);
    dmma(tre[u], ar[u][1], op.bt);
    dmma(tim[u], ai[u][1], op.bt);
    if constexpr (S::TAIL && SFT_CENTRE_DMMA) {
      dmma(csr[u], ar[u][0], op.ts);
      dmma(csi[u], ai[u][0], op.ts);
      dmma(ctr[u], ar[u][1], op.tt);
      dmma(cti[u], ai[u][1], op.tt);
    }
  }
#endif
#pragma unroll
  for (int u = 0; u < NSUB; ++u) {
    // first store: m (sg = 1) or m' (sg = -1), second: the other one
    const double pfr = fma(sg, tre[u][0], sre[u][0]), pfi = fma(sg, tim[u][0], sim[u][0]);  // P = SP +- DP
    const double psr = fma(-sg, tre[u][0], sre[u][0]), psi = fma(-sg, tim[u][0], sim[u][0]);
    const double qfr = fma(sg, sre[u][1], tre[u][1]), qfi = fma(sg, sim[u][1], tim[u][1]);  // Q = SQ +- DQ
    const double qsr = fma(-sg, sre[u][1], tre[u][1]), qsi = fma(-sg, sim[u][1], tim[u][1]);
    if (st_f) {
      o0[u].st(o_f, pfr + qfi, pfi - qfr);  // z_0 = P - iQ
      o1[u].st(o_f, pfr - qfi, pfi + qfr);  // z_1 = P + iQ
    }
    if (st_s) {
      o0[u].st(o_s, psr + qsi, psi - qsr);
      o1[u].st(o_s, psr - qsi, psi + qsr);
    }
  }
  if constexpr (S::TAIL && SFT_CENTRE_DMMA) {
    if (c == 0) {
#pragma unroll
      for (int u = 0; u < NSUB; ++u) {
        // P_H = SP_H, Q_H = SQ_H: z_0 = P - iQ, z_1 = P + iQ
        o0[u].st(H * STR, csr[u][0] + cti[u][0], csi[u][0] - ctr[u][0]);
        o1[u].st(H * STR, csr[u][0] - cti[u][0], csi[u][0] + ctr[u][0]);
      }
    }
  } else if constexpr (S::TAIL) {
    // transpose-reduce over the 4 lanes of a row: lane c ends with component
    // c of (z_0.re, z_0.im, z_1.re, z_1.im) at m = H
    const bool odd = c & 1, hi = c & 2;
#pragma unroll
    for (int u = 0; u < NSUB; ++u) {
      double va = odd ? tl[u][1] : tl[u][0], vb = odd ? tl[u][3] : tl[u][2];
      va += __shfl_xor_sync(0xffffffffu, odd ? tl[u][0] : tl[u][1], 1);
      vb += __shfl_xor_sync(0xffffffffu, odd ? tl[u][2] : tl[u][3], 1);
      double w = hi ? vb : va;
      w += __shfl_xor_sync(0xffffffffu, hi ? va : vb, 2);
      (hi ? o1[u] : o0[u]).st1(H * STR, c & 1, w);
    }
  }
}

// One axis pass of the consumers (NC warps), symmetric form (see SymShape).
// A warp takes super-tiles of 8 fiber tasks: MMA row r (= lane/4) is one
// fiber; lane c = lane%4 loads its fiber's child-0 element 2c+1 and child-1
// element p-2-2c (so s = x_0 + J x_1 and t = x_0 - J x_1 at odd element 2c+1
// are one add each: the A fragments of k = c), and the even pair 2c / p-1-2c
// for the delta columns; 4 DMMA (s and t, real and imaginary parts) give lane
// c the m = c and m' = p-1-c outputs of both children.  Outputs go back in
// place, or to HBM (or a peer's buffer) in the last pass.
// MUL: stage-slot stride of consecutive child slots: 0 = G (slot-major
// stage), 1 for the second level of a two-level tile (transposed slots).
template <int D, int P, int G, int NC, int AX, bool LAST, int LIST = AX, typename E = double2, bool FUSED = false,
          int MUL = 0, bool STAGED = false>
__device__ __forceinline__ void consumer_pass(const TransArgs& a, E* __restrict__ sb,
                                              const unsigned char* __restrict__ blk, const LaneOps<P>& op,
                                              const E* __restrict__ zs, int& rot, int64_t ooff = 0, int round = 0) {
  constexpr int ES = sizeof(E);
  const uint32_t sba = smem_u32(sb), zsa = smem_u32(zs);  // stage and zero slot (shared addresses)
  using S = SymShape<P>;
  using SC = Sched<D, P, G>;
  using ET = ElemT<E>;
  constexpr int H = S::H;
  constexpr int NSUB = NsubCfg<D, P>::v;
  constexpr int PF = Pow<P, D>::v / P;
  constexpr int PD = StrideT<E, Pow<P, D>::v>::v;  // slot stride (elements)
  constexpr int STR = Pow<P, D - 1 - AX>::v;
  constexpr int SH = D - 1 - AX;
  constexpr int C1 = (1 << SH) * (MUL == 0 ? G * PD + SlotPad<D, P, PD>::v : MUL * PD);  // child-1 slot of the pair
  E* const gout = reinterpret_cast<E*>(a.out) + ooff;  // ooff: RHS offset of a batch
  const int* cnt;
  const TaskRec* tasks;
  if constexpr (D == 3) {
    // round `round`, sub-list of axis AX (k = 2 - AX) after the sub-lists of the axes above it
    const int* cr = SC::cnt(blk) + 9 * round;
    int off = 0;
#pragma unroll
    for (int kk = 0; kk < 2 - AX; ++kk) off += cr[3 * kk] + cr[3 * kk + 1] + cr[3 * kk + 2];
    cnt = cr + 3 * (2 - AX);
    tasks = SC::task(blk, round) + off;
  } else {
    cnt = SC::cnt(blk) + 3 * LIST;
    tasks = SC::task(blk, LIST);
  }
  const int ntot = (cnt[0] + cnt[1] + cnt[2]) * PF;
  if (ntot == 0) return;  // (3D: most sub-lists of a round are empty)
  const int nst = (ntot + 7) >> 3;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = lane & 3;
  const int rfib = RowMap<D, P, AX, LAST && !STAGED>::fiber(lane >> 2);  // row -> fiber of the super-tile
  // this lane's element offsets in a fiber (padding k >= H: a valid odd element, zero B row;
  // delta / outputs of lanes c > H (p = 5): clamped, coefficients 0, no stores)
  // (child 1 offsets relative to its own slot)
  const int o_a0 = min(2 * c + 1, P - 2) * STR, o_a1 = max(P - 2 - 2 * c, 1) * STR;
  const int o_d0 = min(2 * c, P - 1) * STR, o_d1 = max(P - 1 - 2 * c, 0) * STR;
  // outputs m = c and m' = p-1-c: one row of each 16-byte-access phase
  // (rows 2q, 2q+1) stores m then m', the other m' then m (role swap, sg =
  // -1); which row swaps depends on the fiber-address step and STR mod 8
  // (SwapEven, from scripts/rfib_model_sym.py) -- with it the phase's loads
  // and stores are bank-conflict free for p = 7 and 3 of 4 instructions for p = 9
  // (a last pass storing straight to HBM keeps one order for all rows: rows
  // 2q, 2q+1 hold consecutive fibers, so one store instruction fills whole
  // 32-byte sectors -- with the swap every sector would be written in two
  // 16-byte halves by two instructions, doubling the L1 -> L2 write sectors)
  const bool swp = !(LAST && !STAGED) && (((lane >> 2) & 1) ^ SwapEven<D, P, AX>::v);
  const double sg = swp ? -1.0 : 1.0;
  const int o_f = (swp ? max(P - 1 - c, H) : min(c, H)) * STR, o_s = (swp ? min(c, H) : max(P - 1 - c, H)) * STR;
  const bool st_f = c <= H, st_s = c < H;
  // units of NSUB super-tiles go round-robin over the warps, continuing from
  // where the previous pass stopped (rot), so that the extra unit of a pass
  // whose count is not a multiple of NC does not always land on warp 0
  const int j0 = warp >= rot ? warp - rot : warp - rot + NC;
  // (measured: C2 -0.8%, C1 -2%, C3 +2%: 2D only)
  if (SFT_ROTATE && (D == 2 || SFT_ROTATE3)) rot = (rot + (nst + NSUB - 1) / NSUB) % NC;
  for (int st0 = j0 * NSUB; st0 < nst; st0 += NC * NSUB) {
    // child slots of the row's pair; an absent child (its task's class bit
    // clear) reads the CTA's zero slot instead: absent slots are never
    // zero-filled or read
    // STAGED: the last pass also writes in place; the tile's outputs then
    // leave the stage by TMA bulk stores (tma_store_tile)
    constexpr bool GL = LAST && !STAGED;
    uint32_t xa[NSUB], xb[NSUB];
    OutRow<E, GL> o0[NSUB], o1[NSUB];
    unsigned orc = 0;  // classes of this lane's rows
#pragma unroll
    for (int u = 0; u < NSUB; ++u) {
      const int tau = (st0 + u) * 8 + rfib;
      const bool vrow = tau < ntot;
      TaskRec d;
      int ebase = 0;
      if (vrow) {
        d = tasks[tau / PF];
        const int f = tau % PF;
        ebase = (f / STR) * STR * P + f % STR;
      } else {
        d.x = 0;
        d.cls = 0;
        d.o0 = d.o1 = ~0u;
      }
      const uint32_t xo = d.x + (uint32_t)ebase;
      orc |= d.cls;
#if SFT_ABSENT == 2
      xa[u] = (d.cls & 1u) ? sba + xo * ES : zsa + ebase * ES;
      xb[u] = (d.cls & 2u) ? sba + (xo + C1) * ES : zsa + ebase * ES;
#else  // zero-filled absent slots
      xa[u] = sba + xo * ES;
      xb[u] = sba + (xo + C1) * ES;
#endif

      o0[u].g = o1[u].g = nullptr;
      o0[u].s = sba + xo * ES;
      o1[u].s = sba + (xo + C1) * ES;
#ifdef SFT_ABL_NOSTORE  // ablation: no output stores (shared or global)
      o0[u].ok = o1[u].ok = false;
#else
      if (GL && FUSED) {
        // fused exchange: straight into the receiving rank's buffer
        auto dst = [&](uint32_t off) -> E* {
          if (off == ~0u) return nullptr;
          const int64_t i = (int64_t)(off / (uint32_t)PD);
          int q = 0;
          while (q + 1 < a.npeer && i >= a.peer_seg[q + 1]) ++q;
          return reinterpret_cast<E*>(a.peer[q]) + a.peer_off[q] + (i - a.peer_seg[q]) * PD + ebase;
        };
        o0[u].g = dst(d.o0);
        o1[u].g = dst(d.o1);
        o0[u].ok = o0[u].g != nullptr;
        o1[u].ok = o1[u].g != nullptr;
      } else if (GL) {
        o0[u].g = gout + d.o0 + ebase;
        o1[u].g = gout + d.o1 + ebase;
        o0[u].ok = d.o0 != ~0u;
        o1[u].ok = d.o1 != ~0u;
      } else {
        o0[u].ok = o1[u].ok = vrow;
      }
#endif
    }
    // warp-uniform union of the rows' child classes: super-tiles whose rows
    // all lack one child skip its loads (the task lists are class-sorted, so
    // most super-tiles are class-uniform)
    const unsigned pres = (SFT_CLASS_SPLIT && ((D == 2 && UseSym<P>::v) || (D == 3 && SFT_CLASS_SPLIT3))) ? __reduce_or_sync(0xffffffffu, orc) : 3u;
    if constexpr (!UseSym<P>::v) {
      if (pres == 1u) direct_math<D, P, STR, C1, NSUB, E, GL, 1>(op, xa, xb, o0, o1, c);
      else if (pres == 2u) direct_math<D, P, STR, C1, NSUB, E, GL, 2>(op, xa, xb, o0, o1, c);
      else direct_math<D, P, STR, C1, NSUB, E, GL, 3>(op, xa, xb, o0, o1, c);
    } else {
      if (pres == 1u)
        sym_math<D, P, STR, C1, NSUB, E, GL, 1>(op, xa, xb, o0, o1, c, o_a0, o_a1, o_d0, o_d1, o_f, o_s, st_f, st_s, sg);
      else if (pres == 2u)
        sym_math<D, P, STR, C1, NSUB, E, GL, 2>(op, xa, xb, o0, o1, c, o_a0, o_a1, o_d0, o_d1, o_f, o_s, st_f, st_s, sg);
      else
        sym_math<D, P, STR, C1, NSUB, E, GL, 3>(op, xa, xb, o0, o1, c, o_a0, o_a1, o_d0, o_d1, o_f, o_s, st_f, st_s, sg);
    }
  }
  // staged last pass: this thread's stage writes before the async-proxy
  // (TMA) reads of the bulk stores
  if constexpr (LAST && STAGED) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// TMA store of a tile whose last pass ran in place (STAGED): every output
// array (A-child alpha of a group's A', B) is one contiguous p^d array in the
// stage and in HBM, so one 1-D bulk copy shared -> global each (lanes of one
// warp issue a task's two outputs each), instead of per-lane 16-byte global
// stores from registers.  Returns after the copies have read the stage (the
// caller then releases it to the producer).
// Measured (B200, same box): C2 translate 1.017 (1) vs 0.953 ms (0), C4 35.4 vs
// 34.4 ms -- the extra barrier and the serial issue cost more than the per-lane
// stores, once those fill whole sectors (see consumer_pass); off by default.
#ifndef SFT_TMA_STORE
#define SFT_TMA_STORE 0
#endif
template <int D, int P, int G, typename E>
__device__ __forceinline__ void tma_store_tile(const TransArgs& a, const unsigned char* __restrict__ blk, const E* sb,
                                               int64_t ooff) {
  using SC = Sched<D, P, G>;
  constexpr int PS = StrideT<E, Pow<P, D>::v>::v;
  constexpr uint32_t BYTES = PS * (uint32_t)sizeof(E);
  const int lane = threadIdx.x & 31;
  E* const out = reinterpret_cast<E*>(a.out) + ooff;
  const uint32_t sba = smem_u32(sb);
  auto bulk = [&](const E* dst, uint32_t src) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(BYTES)
                 : "memory");
  };
  static_assert(D == 2, "staged last pass: 2D only");
#pragma unroll
  for (int li = 0; li < 2; ++li) {
    // last-pass lists: 0 (axis 0: child slots (1 << (d-1)) G arrays apart), 3 (2D reversed order: axis 1, G apart)
    const int L = li == 0 ? 0 : 3;
    const uint32_t C1 = (uint32_t)((li == 0 ? (1 << (D - 1)) : 1) * (G * PS + SlotPad<D, P, PS>::v));
    const int* cnt = SC::cnt(blk) + 3 * L;
    const int n = cnt[0] + cnt[1] + cnt[2];
    const TaskRec* tk = SC::task(blk, L);
    for (int t = lane; t < n; t += 32) {
      const TaskRec r = tk[t];
      if (r.o0 != ~0u) bulk(out + r.o0, sba + r.x * (uint32_t)sizeof(E));
      if (r.o1 != ~0u) bulk(out + r.o1, sba + (r.x + C1) * (uint32_t)sizeof(E));
    }
  }
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
  asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  __syncwarp();
}

// Optional cycle accounting (-DSFT_INSTR): per-CTA sums of clock64 intervals
// into g_instr[blockIdx][8]: 0 producer total, 1 producer wait(empty),
// 2 producer issue, 3 consumer total, 4 consumer wait(full),
// 5 consumer first pass(es), 6 consumer wait before the last pass, 7 consumer last pass.
#ifdef SFT_INSTR
__device__ unsigned long long* g_instr = nullptr;
#define INSTR_T0(v) const long long v = clock64()
#define INSTR_ADD(k, t0)                                                                      \
  do {                                                                                        \
    if ((threadIdx.x & 31) == 0 && g_instr)                                                   \
      atomicAdd(&g_instr[(size_t)blockIdx.x * 8 + (k)], (unsigned long long)(clock64() - (t0))); \
  } while (0)
#else
#define INSTR_T0(v)
#define INSTR_ADD(k, t0)
#endif

// named barrier over the NT consumer threads (the producer warp never joins)
template <int NT>
__device__ __forceinline__ void consumer_sync() {
#ifdef SFT_ABL_NOBAR  // ablation: no pass barrier (wrong results; timing only)
  __syncwarp();
#else
  asm volatile("bar.sync 1, %0;" ::"n"(NT) : "memory");
#endif
}

#ifndef SFT_PRODUCER_SLEEP
#define SFT_PRODUCER_SLEEP 200  // ns between the producer's polls of a stage's empty barrier
#endif
__device__ __forceinline__ void mbar_wait_sleep(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (true) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
    if (done) break;
    if (SFT_PRODUCER_SLEEP > 0) __nanosleep(SFT_PRODUCER_SLEEP);
  }
}

// Producer warp of the warp-specialised kernels: runs up to NST tiles ahead;
// per tile arms full[s] with the byte count, bulk-copies the tile's schedule
// block into blk[s] and every present child array into stage s (reading the
// group records of its next tile from HBM while it waits for a free stage).
// Issue one tile (work item w = tile * nrhs + r) into stage s, by one whole
// warp: zero the slots of absent children (the consumers read every slot
// unmasked), arm full[s] with the byte count, bulk-copy (1-D TMA) the tile's
// schedule block and every present child array.  gr = this lane's group
// record (first child pair index, child mask) for lane < G.
// NB: schedule blocks per tile (2 for a two-level tile: one per level)
// nrec_src / nrec_dst (producer-less kernels): also bulk-copy the group
// records of the work item that will next use this stage (the tile's stage
// refill then needs no HBM read of its own), nrec_src = nullptr: none.
template <int D, int P, int G, int NST, typename E, int PS, bool BATCH, int NB = 1>
__device__ __forceinline__ void ws_issue(const TransArgs& a, const unsigned char* __restrict__ sched, int64_t w,
                                         int64_t tile, uint2 gr, E* ring,
                                         unsigned char (*blk)[Sched<D, P, G>::BLK * NB], uint64_t* full, int s,
                                         int64_t* wid, const unsigned char* nrec_src = nullptr, uint32_t nrec_dst = 0) {
  using SC = Sched<D, P, G>;
  constexpr int PD = PS;  // stage and HBM arrays have stride PS elements of type E
  constexpr int NS = 1 << D;
  constexpr int STAGE = NS * (G * PD + SlotPad<D, P, PD>::v);
  const int lane = threadIdx.x & 31;
  const int64_t nr = BATCH ? a.nrhs : 1;
  const E* const ain = reinterpret_cast<const E*>(a.in) + (BATCH ? (w - tile * nr) * a.rs : (int64_t)0);
  uint32_t nbytes = __popc(gr.y) * PD * (uint32_t)sizeof(E);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nbytes += __shfl_xor_sync(0xffffffffu, nbytes, o);
  E* sb = ring + s * STAGE;
  // uniform tile: G groups of one B with consecutive A' (the common case) --
  // every child slot's G arrays are contiguous in HBM and in the slot-major
  // stage, so one bulk copy per present child slot.  Absent children's slots
  // are not touched: the consumers read only the slots their task's class
  // marks present.
  const int ng = (int)min((int64_t)G, a.ngroups - tile * G);
  const uint32_t m0 = __shfl_sync(0xffffffffu, gr.y, 0), p0 = __shfl_sync(0xffffffffu, gr.x, 0);
  const bool mine_ok = lane >= G || (gr.y == m0 && gr.x == p0 + (uint32_t)lane);
  const bool uniform = __all_sync(0xffffffffu, mine_ok) && ng == G && m0 != 0u;
#if SFT_ABSENT == 0
  {
    constexpr int CH = PD * (int)sizeof(E) / 16;  // 16-byte chunks per slot
    if (uniform) {
      for (int c = 0; c < NS; ++c) {
        if (m0 >> c & 1) continue;
        float4* z = reinterpret_cast<float4*>(sb + (int64_t)c * (G * PD + SlotPad<D, P, PD>::v));
        for (int q = lane; q < G * CH; q += 32) z[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    } else {
      for (int js = 0; js < ng * NS; ++js) {
        const int j = js / NS, c = js % NS;
        const uint32_t mB = __shfl_sync(0xffffffffu, gr.y, j);
        if (mB >> c & 1) continue;
        float4* z = reinterpret_cast<float4*>(sb + (int64_t)c * (G * PD + SlotPad<D, P, PD>::v) + (int64_t)j * PD);
        for (int q = lane; q < CH; q += 32) z[q] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
  }
#endif
  // the consumers' generic-proxy accesses of this stage (released through
  // empty[s]) are ordered before the async-proxy writes below
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncwarp();
  if (lane == 0) {
    wid[s] = w;  // the consumers read the stage's work item after full[s] (arrive: release)
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                 "r"(nbytes + (uint32_t)(SC::BLK * NB) + (nrec_src ? (uint32_t)SC::GRP : 0u))
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(&blk[s][0])),
        "l"(sched + tile * (SC::BLK * NB)), "r"((uint32_t)(SC::BLK * NB)), "r"(smem_u32(&full[s]))
        : "memory");
    if (nrec_src)
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(nrec_dst),
          "l"(nrec_src), "r"((uint32_t)SC::GRP), "r"(smem_u32(&full[s]))
          : "memory");
  }
  __syncwarp();
  if (uniform) {
    // lane c < NS: child slot c of all G groups, one copy of G arrays
    if (lane < NS && (m0 >> lane & 1)) {
      const int r = __popc(m0 & ((1u << lane) - 1u));
      const int64_t pin = (int64_t)p0 + (int64_t)r * a.in_nA;
#ifndef SFT_ABL_NOLOAD
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              smem_u32(sb + (int64_t)lane * (G * PD + SlotPad<D, P, PD>::v))),
          "l"(ain + pin * PD), "r"((uint32_t)(G * PD * sizeof(E))), "r"(smem_u32(&full[s]))
          : "memory");
#else
      (void)pin;
      asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])),
                   "r"((uint32_t)(G * PD * sizeof(E)))
                   : "memory");
#endif
    }
    return;
  }
  uint32_t mm = gr.y;
  int r = 0;
  while (mm) {
    const int c = __ffs(mm) - 1;
    mm &= mm - 1;
    const int64_t pin = (int64_t)gr.x + (int64_t)(r++) * a.in_nA;
#ifndef SFT_ABL_NOLOAD
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(sb + (int64_t)c * (G * PD + SlotPad<D, P, PD>::v) + (int64_t)lane * PD)),
        "l"(ain + pin * PD), "r"((uint32_t)(PD * sizeof(E))), "r"(smem_u32(&full[s]))
        : "memory");
#else
    (void)pin;
    asm volatile("mbarrier.complete_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])),
                 "r"((uint32_t)(PD * sizeof(E)))
                 : "memory");
#endif
  }
}

template <int D, int P, int G, int NB = 1>
__device__ __forceinline__ uint2 ws_group_record(const unsigned char* __restrict__ sched, int64_t tile, bool ok) {
  using SC = Sched<D, P, G>;
  const int lane = threadIdx.x & 31;
  return (ok && lane < G) ? __ldg(reinterpret_cast<const uint2*>(sched + tile * (SC::BLK * NB) + SC::HDR) + lane)
                          : make_uint2(0u, 0u);
}

template <int D, int P, int G, int NST, typename E = double2, int PS = StrideT<double2, Pow<P, D>::v>::v, bool BATCH = false, int NB = 1>
__device__ __forceinline__ void ws_producer(const TransArgs& a, const unsigned char* __restrict__ sched, int64_t ntiles,
                                            E* ring, unsigned char (*blk)[Sched<D, P, G>::BLK * NB], uint64_t* full,
                                            uint64_t* empty, int64_t* wid) {
  INSTR_T0(tp0);
  int s = 0;
  uint32_t ph = 0;
  // work items w = tile * nrhs + r (BATCH = false: nrhs = 1, w = tile)
  const int64_t nr = BATCH ? a.nrhs : 1;
  const int64_t nwork = ntiles * nr;
  const int lane = threadIdx.x & 31;
  // next work item: dynamic (a shared counter, one fetch ahead) or grid-stride
  auto fetch = [&](int64_t cur) -> int64_t {
    if (!a.ctr) return cur + gridDim.x;
    int v = 0;
    if (lane == 0) v = atomicAdd(&a.ctr[0], 1);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  int64_t w = a.ctr ? fetch(0) : (int64_t)blockIdx.x;
  int64_t tile = BATCH ? w / nr : w;
  uint2 gr = ws_group_record<D, P, G, NB>(sched, tile, w < nwork);
  // programmatic dependent launch: everything above (schedule reads, barrier
  // init, the consumers' operand loads) overlaps the previous level's tail;
  // the previous level's output (our input) and input (our output buffer)
  // are touched only after it has completed
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // (after the wait: see launch_pdl)
  int i = 0;
  for (; w < nwork; ++i) {
    const int64_t wn = fetch(w);
    const int64_t next = BATCH ? wn / nr : wn;
    const uint2 gn = ws_group_record<D, P, G, NB>(sched, next, wn < nwork);
    INSTR_T0(tw0);
    if (i >= NST) mbar_wait_sleep(smem_u32(&empty[s]), ph ^ 1u);
    INSTR_ADD(1, tw0);
    INSTR_T0(tb0);
    ws_issue<D, P, G, NST, E, PS, BATCH, NB>(a, sched, w, tile, gr, ring, blk, full, s, wid);
    INSTR_ADD(2, tb0);
    gr = gn;
    w = wn;
    tile = next;
    if (++s == NST) {
      s = 0;
      ph ^= 1u;
    }
  }
  // end of work: a sentinel item (-1) in the next stage of the sequence
  if (i >= NST) mbar_wait_sleep(smem_u32(&empty[s]), ph ^ 1u);
  if (lane == 0) {
    wid[s] = -1;
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
    // dynamic scheduling: the last CTA done fetching resets the counters for
    // the next apply (every CTA's final fetch precedes its increment here)
    if (a.ctr) {
      __threadfence();
      if (atomicAdd(&a.ctr[1], 1) == (int)gridDim.x - 1) {
        a.ctr[0] = 0;
        a.ctr[1] = 0;
      }
    }
  }
  INSTR_ADD(0, tp0);
}

// Warp-specialised translation kernel (default).  Warp NC is the producer: it
// runs up to NST tiles ahead, and per tile arms full[s] with the byte count,
// bulk-copies the tile's schedule block into the stage bookkeeping and every
// present child array into the stage (reading the group records of its next
// tile from HBM while it waits for a free stage).  Warps 0..NC-1 consume.
// 2D with NST >= 3: skewed pipeline, pass 1 of tile i+1 runs before pass 0 of
// tile i, and pass 0 waits on an mbarrier (p1done) every consumer thread
// arrives on after its pass-1 rows, so warps do not idle at a pass barrier.
//
// PL (producer-less, SFT_PL=1; measured slower, off): no producer warp -- all NC warps consume; warp 0
// issues the first NST tiles, and afterwards the last consumer warp to finish
// a tile (smem counter done[s]) refills its stage with the work item NST
// grid-strides ahead.  The group records that refill needs arrived in the
// stage bookkeeping (nrec[s]) with the tile's own loads, so it reads no HBM.
// Same threads per CTA as NC - 1 consumers + a producer, one more consumer.
template <int D, int P, int G, int NC, int NST, int MINB, typename E = double2, bool FUSED = false,
          bool BATCH = false, bool F2 = false, bool PL = false>
__global__ __launch_bounds__((NC + (PL ? 0 : 1)) * 32, MINB) void k_translate_ws(TransArgs a,
                                                                                  const double* __restrict__ frag,
                                                                                  const unsigned char* __restrict__ sched,
                                                                                  int64_t ntiles) {
  static_assert(!F2 || (D == 2 && NST < 3 && G % 4 == 0 && !FUSED), "two-level tiles: 2D, unskewed, G = 4k");
  using SC = Sched<D, P, G>;
  constexpr int PD = StrideT<E, Pow<P, D>::v>::v;  // array stride (elements)
  constexpr int NS = 1 << D;
  constexpr int STAGE = NS * (G * PD + SlotPad<D, P, PD>::v);
  extern __shared__ __align__(128) unsigned char smem_raw[];
  E* ring = reinterpret_cast<E*>(smem_raw);  // [NST][G][NS][PD]
  E* const zs = ring + NST * STAGE;          // [PD] zeros: what an absent child slot reads
  constexpr int NB = F2 ? 2 : 1;  // schedule blocks per tile
  __shared__ __align__(128) unsigned char blk[NST][SC::BLK * NB];
  __shared__ __align__(8) uint64_t full[NST], empty[NST], p1done[NST];
  __shared__ __align__(8) uint64_t r1done[D == 3 && NST >= 3 ? NST : 1];  // 3D skewed: round 1 of the stage done
  __shared__ __align__(16) unsigned char nrec[PL ? NST : 1][SC::GRP];  // PL: group records of the stage's next item
  __shared__ int done[NST];                                            // PL: consumer warps done with the stage
  __shared__ int64_t wid[NST];  // work item in each stage (-1: no more work)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x < NST) {
    done[threadIdx.x] = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[threadIdx.x])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[threadIdx.x])), "r"(NC));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&p1done[threadIdx.x])), "r"(NC * 32));
    if constexpr (D == 3 && NST >= 3)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&r1done[threadIdx.x])), "r"(NC * 32));
  }
  if (threadIdx.x == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  for (int q = threadIdx.x; q < PD * (int)sizeof(E) / 16; q += blockDim.x)
    reinterpret_cast<float4*>(zs)[q] = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncthreads();
  if constexpr (!PL) {
    if (warp == NC) {
      ws_producer<D, P, G, NST, E, PD, BATCH, NB>(a, sched, ntiles, ring, blk, full, empty, wid);
      return;
    }
  }
  // ---------------- consumers ----------------
  LaneOps<P> op;
  load_lane_ops(op, frag, lane);
  // every thread waits for the previous level before it triggers the next
  // one's launch (the consumers would wait for the stage anyway)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t nr_ = BATCH ? a.nrhs : 1;
  const int64_t nwork_ = ntiles * nr_;
  // PL: issue work item w into stage s (one whole warp), with the group
  // records of item w + NST * grid (the stage's next item) when it exists
  auto pl_issue = [&](int64_t w, uint2 gr, int st) {
    const int64_t wn = w + (int64_t)NST * gridDim.x;
    const unsigned char* nsrc =
        wn < nwork_ ? sched + (BATCH ? wn / nr_ : wn) * (int64_t)(SC::BLK * NB) + SC::HDR : nullptr;
    ws_issue<D, P, G, NST, E, PD, BATCH, NB>(a, sched, w, BATCH ? w / nr_ : w, gr, ring, blk, full, st, wid, nsrc,
                                             smem_u32(&nrec[PL ? st : 0][0]));
  };
  // PL: no more work for stage st -- the sentinel item
  auto pl_end = [&](int st) {
    if (lane == 0) {
      wid[st] = -1;
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[st])) : "memory");
    }
  };
  if constexpr (PL) {
    if (warp == 0) {
      for (int i = 0; i < NST; ++i) {
        const int64_t w = blockIdx.x + (int64_t)i * gridDim.x;
        if (w >= nwork_) {
          pl_end(i);
          break;
        }
        pl_issue(w, ws_group_record<D, P, G, NB>(sched, BATCH ? w / nr_ : w, true), i);
      }
    }
  }
  // a consumer warp is done with the item w in stage st: PL -- the last warp
  // to get here refills the stage; otherwise release it to the producer
  auto release = [&](int64_t w, int st) {
    __syncwarp();
    if constexpr (PL) {
      int last = 0;
      if (lane == 0) {
        int old;
        asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(&done[st])) : "memory");
        last = old == NC - 1;
        if (last) done[st] = 0;
      }
      last = __shfl_sync(0xffffffffu, last, 0);
      if (last) {
        const int64_t wn = w + (int64_t)NST * gridDim.x;
        if (wn < nwork_) {
          const uint2 gr = lane < G ? reinterpret_cast<const uint2*>(&nrec[PL ? st : 0][0])[lane] : make_uint2(0u, 0u);
          pl_issue(wn, gr, st);
        } else {
          pl_end(st);
        }
      }
    } else {
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[st])) : "memory");
    }
  };
  int s = 0, rot = 0;
  uint32_t ph = 0;
  INSTR_T0(tc0);
  // 2D: first passes (list 1: axis 1, list 2: axis 0 for groups in reversed
  // order), then last passes (list 0: axis 0, list 3: axis 1)
  auto first2d = [&](E* sb_, const unsigned char* bk) {
    consumer_pass<D, P, G, NC, D - 1, false, 1, E>(a, sb_, bk, op, zs, rot, 0);
    if constexpr (D == 2) consumer_pass<D, P, G, NC, 0, false, 2, E>(a, sb_, bk, op, zs, rot, 0);
  };
  auto last2d = [&](E* sb_, const unsigned char* bk, int64_t oo) {
    consumer_pass<D, P, G, NC, 0, true, 0, E, FUSED>(a, sb_, bk, op, zs, rot, oo);
    if constexpr (D == 2) consumer_pass<D, P, G, NC, D - 1, true, 3, E, FUSED>(a, sb_, bk, op, zs, rot, oo);
  };
  // work items w = tile * nrhs + r; the output of RHS r goes to out + r * rs
  auto ooff = [&](int64_t w_) { return BATCH ? (w_ % a.nrhs) * a.rs : (int64_t)0; };
  // the last pass in place + TMA bulk stores (non-skewed single-level tiles)
  constexpr bool STAGE_OUT = SFT_TMA_STORE && !FUSED && !F2 && D == 2;  // (2D only)
  // the work item of each stage comes from the producer (wid, after full[s]);
  // -1 ends the sequence (dynamic or grid-stride assignment alike)
  // 3D round r of the tile in stage sb: the axis-2, -1, -0 sub-lists (r < 2 in
  // place, r = 2 to HBM)
  auto round3 = [&](E* sb_, const unsigned char* bk, int r, int64_t oo) {
    if constexpr (D == 3) {
      if (r < 2) {
        consumer_pass<D, P, G, NC, 2, false, 0, E>(a, sb_, bk, op, zs, rot, 0, r);
        consumer_pass<D, P, G, NC, 1, false, 0, E>(a, sb_, bk, op, zs, rot, 0, r);
        consumer_pass<D, P, G, NC, 0, false, 0, E>(a, sb_, bk, op, zs, rot, 0, r);
      } else {
        consumer_pass<D, P, G, NC, 2, true, 0, E, FUSED>(a, sb_, bk, op, zs, rot, oo, 2);
        consumer_pass<D, P, G, NC, 1, true, 0, E, FUSED>(a, sb_, bk, op, zs, rot, oo, 2);
        consumer_pass<D, P, G, NC, 0, true, 0, E, FUSED>(a, sb_, bk, op, zs, rot, oo, 2);
      }
    }
  };
  if constexpr (D == 3 && NST >= 3 && !F2) {
    // 3D skewed pipeline: per tile i, round 1 of i, round 0 of i+1, round 2
    // of i -- each round's dependency (the previous round of the same tile, on
    // every warp: p1done = round 0 done, r1done = round 1 done) is waited on
    // one round of other work later, so warps do not idle at pass barriers
    mbar_wait(smem_u32(&full[0]), 0);
    int64_t tile = wid[0];
    if (tile >= 0) {
      round3(ring, blk[0], 0, 0);
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&p1done[0])) : "memory");
    }
    while (tile >= 0) {
      const int sn = s + 1 == NST ? 0 : s + 1;
      const uint32_t phn = sn == 0 ? ph ^ 1u : ph;
      E* const sb = ring + s * STAGE;
      mbar_wait(smem_u32(&p1done[s]), ph);
      round3(sb, blk[s], 1, 0);
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&r1done[s])) : "memory");
      mbar_wait(smem_u32(&full[sn]), phn);
      const int64_t nt = wid[sn];
      if (nt >= 0) {
        round3(ring + sn * STAGE, blk[sn], 0, 0);
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&p1done[sn])) : "memory");
      }
      mbar_wait(smem_u32(&r1done[s]), ph);
      round3(sb, blk[s], 2, ooff(tile));
      release(tile, s);
      s = sn;
      ph = phn;
      tile = nt;
    }
  } else if constexpr (D == 2 && NST >= 3 && !F2) {
    mbar_wait(smem_u32(&full[0]), 0);
    int64_t tile = wid[0];
    if (tile >= 0) {
      first2d(ring, blk[0]);
      asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&p1done[0])) : "memory");
    }
    while (tile >= 0) {
      const int sn = s + 1 == NST ? 0 : s + 1;
      const uint32_t phn = sn == 0 ? ph ^ 1u : ph;
      INSTR_T0(tf0);
      mbar_wait(smem_u32(&full[sn]), phn);
      INSTR_ADD(4, tf0);
      const int64_t nt = wid[sn];
      if (nt >= 0) {
        INSTR_T0(t1);
        first2d(ring + sn * STAGE, blk[sn]);
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&p1done[sn])) : "memory");
        INSTR_ADD(5, t1);
      }
      INSTR_T0(t2);
      mbar_wait(smem_u32(&p1done[s]), ph);
      INSTR_ADD(6, t2);
      INSTR_T0(t3);
      last2d(ring + s * STAGE, blk[s], ooff(tile));
      INSTR_ADD(7, t3);
      release(tile, s);
      s = sn;
      ph = phn;
      tile = nt;
    }
  } else {
    for (;;) {
      INSTR_T0(tf0);
      mbar_wait(smem_u32(&full[s]), ph);
      INSTR_ADD(4, tf0);
      const int64_t w = wid[s];
      if (w < 0) break;
      E* sb = ring + s * STAGE;
      if constexpr (F2) {
        // two-level tile: first level (block 0) in place, second level (block
        // 1) on the transposed slots, its second pass to HBM
        const unsigned char* bk0 = blk[s];
        const unsigned char* bk1 = blk[s] + SC::BLK;
        INSTR_T0(t1);
        consumer_pass<D, P, G, NC, 1, false, 1, E>(a, sb, bk0, op, zs, rot, 0);
        consumer_pass<D, P, G, NC, 0, false, 2, E>(a, sb, bk0, op, zs, rot, 0);
        INSTR_ADD(5, t1);
        INSTR_T0(t2);
        consumer_sync<NC * 32>();
        INSTR_ADD(6, t2);
        INSTR_T0(t3);
        consumer_pass<D, P, G, NC, 0, false, 0, E>(a, sb, bk0, op, zs, rot, 0);
        consumer_pass<D, P, G, NC, 1, false, 3, E>(a, sb, bk0, op, zs, rot, 0);
        INSTR_ADD(5, t3);
        INSTR_T0(t4);
        consumer_sync<NC * 32>();
        INSTR_ADD(6, t4);
        INSTR_T0(t5);
        consumer_pass<D, P, G, NC, 1, false, 1, E, false, 1>(a, sb, bk1, op, zs, rot, 0);
        consumer_pass<D, P, G, NC, 0, false, 2, E, false, 1>(a, sb, bk1, op, zs, rot, 0);
        INSTR_ADD(7, t5);
        INSTR_T0(t6);
        consumer_sync<NC * 32>();
        INSTR_ADD(6, t6);
        INSTR_T0(t7);
        consumer_pass<D, P, G, NC, 0, true, 0, E, false, 1>(a, sb, bk1, op, zs, rot, ooff(w));
        consumer_pass<D, P, G, NC, 1, true, 3, E, false, 1>(a, sb, bk1, op, zs, rot, ooff(w));
        INSTR_ADD(7, t7);
      } else if constexpr (D == 2) {
        INSTR_T0(t1);
        first2d(sb, blk[s]);
        INSTR_ADD(5, t1);
        INSTR_T0(t2);
        consumer_sync<NC * 32>();
        INSTR_ADD(6, t2);
        INSTR_T0(t3);
        if constexpr (STAGE_OUT) {
          consumer_pass<D, P, G, NC, 0, true, 0, E, false, 0, true>(a, sb, blk[s], op, zs, rot, 0);
          consumer_pass<D, P, G, NC, D - 1, true, 3, E, false, 0, true>(a, sb, blk[s], op, zs, rot, 0);
          consumer_sync<NC * 32>();
          if (warp == 0) tma_store_tile<D, P, G, E>(a, blk[s], sb, ooff(w));
        } else {
          last2d(sb, blk[s], ooff(w));
        }
        INSTR_ADD(7, t3);
      } else {
        // 3D: rounds 0, 1 in place, round 2 to HBM; in each round every group
        // runs the pass of its own order's axis (sub-lists of axes 2, 1, 0)
#if SFT_ROUND_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
        for (int r = 0; r < 2; ++r) {
          consumer_pass<D, P, G, NC, 2, false, 0, E>(a, sb, blk[s], op, zs, rot, 0, r);
          consumer_pass<D, P, G, NC, 1, false, 0, E>(a, sb, blk[s], op, zs, rot, 0, r);
          consumer_pass<D, P, G, NC, 0, false, 0, E>(a, sb, blk[s], op, zs, rot, 0, r);
          consumer_sync<NC * 32>();
        }
        consumer_pass<D, P, G, NC, 2, true, 0, E, FUSED>(a, sb, blk[s], op, zs, rot, ooff(w), 2);
        consumer_pass<D, P, G, NC, 1, true, 0, E, FUSED>(a, sb, blk[s], op, zs, rot, ooff(w), 2);
        consumer_pass<D, P, G, NC, 0, true, 0, E, FUSED>(a, sb, blk[s], op, zs, rot, ooff(w), 2);
      }
      release(w, s);
      if (++s == NST) {
        s = 0;
        ph ^= 1u;
      }
    }
  }
  // bulk stores complete before the CTA exits (the next level reads them)
  if (warp == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  // fused exchange: make this rank's peer stores visible system-wide before
  // the kernel completes (the caller's cross-rank barrier follows on the stream)
  if (FUSED) __threadfence_system();
  INSTR_ADD(3, tc0);
}

// Per-lane operator table of the symmetric pass (SymShape), built from the
// long-double host tables of beta = 0 (RC_0, RS_0).  Returns {} (an error) if
// the tables lack the mirror symmetry or the delta structure the kernel's
// split relies on (never for p = 5, 7, 9).
template <int P>
static std::vector<double> sym_fragments() {
  using S = SymShape<P>;
  constexpr int H = S::H;
  std::vector<double> V, invD, RC, RS;
  build_tables_host(P, V, invD, &RC, &RS);
  auto rc = [&](int b, int m, int l) { return RC[((size_t)b * P + m) * P + l]; };
  auto rs = [&](int b, int m, int l) { return RS[((size_t)b * P + m) * P + l]; };
  // mirror symmetry RC_1 = J RS_0 J, RS_1 = J RC_0 J
  for (int m = 0; m < P; ++m)
    for (int l = 0; l < P; ++l)
      if (std::fabs(rc(1, m, l) - rs(0, P - 1 - m, P - 1 - l)) > 1e-15 ||
          std::fabs(rs(1, m, l) - rc(0, P - 1 - m, P - 1 - l)) > 1e-15)
        return {};
  // column n of the s- / t-GEMM at element l (the 1/2 of the sum/difference folded in)
  auto col = [&](bool tg, int n, int l) -> double {
    const int m = n / 2, mp = P - 1 - m;
    if (m < H) {
      if (!tg) return n % 2 == 0 ? 0.5 * (rc(0, m, l) + rc(0, mp, l)) : 0.5 * (rs(0, m, l) - rs(0, mp, l));
      return n % 2 == 0 ? 0.5 * (rc(0, m, l) - rc(0, mp, l)) : 0.5 * (rs(0, m, l) + rs(0, mp, l));
    }
    if (m == H && !S::TAIL) return tg ? (n % 2 == 1 ? rs(0, H, l) : 0.0) : (n % 2 == 0 ? rc(0, H, l) : 0.0);
    return 0.0;
  };
  std::vector<double> fr(S::NFRAG, 0.0);
  for (int lane = 0; lane < 32; ++lane) {
    const int k = lane & 3, n = lane >> 2, c = lane & 3;
    fr[S::OFF_BS + lane] = k < H ? col(false, n, 2 * k + 1) : 0.0;
    fr[S::OFF_BT + lane] = k < H ? col(true, n, 2 * k + 1) : 0.0;
    const bool ev = 2 * c <= P - 1;
    fr[S::OFF_DS + lane] = ev ? col(false, 2 * c, 2 * c) : 0.0;
    fr[S::OFF_DS + 32 + lane] = ev ? col(false, 2 * c + 1, 2 * c) : 0.0;
    fr[S::OFF_DT + lane] = ev ? col(true, 2 * c, 2 * c) : 0.0;
    fr[S::OFF_DT + 32 + lane] = ev ? col(true, 2 * c + 1, 2 * c) : 0.0;
    // the split is exact only if lane c's columns have no other even entries
    for (int i = 0; 2 * i <= P - 1; ++i)
      if (i != c)
        for (int nn = 2 * c; nn <= 2 * c + 1; ++nn)
          if (col(false, nn, 2 * i) != 0.0 || col(true, nn, 2 * i) != 0.0) return {};
    if (S::TAIL) {
      // centre tile B fragments (column n = 0 only) or the tail's per-lane k weights
      const bool live = k < H && (!SFT_CENTRE_DMMA || n == 0);
      fr[S::OFF_TAIL + lane] = live ? rc(0, H, 2 * k + 1) : 0.0;
      fr[S::OFF_TAIL + 32 + lane] = live ? rs(0, H, 2 * k + 1) : 0.0;
      fr[S::OFF_TAIL + 64 + lane] = c == 0 ? rc(0, H, P - 1) : 0.0;
      fr[S::OFF_TAIL + 96 + lane] = c == 0 ? rs(0, H, P - 1) : 0.0;
    }
  }
  if (S::TAIL)
    for (int i = 0; 2 * i < P - 1; ++i)
      if (rc(0, H, 2 * i) != 0.0 || rs(0, H, 2 * i) != 0.0) return {};
  return fr;
}

// Per-lane table of the direct form (p = 5): stacked K = (child 0: elements
// 1, 3; child 1: elements 1, 3), columns (P_m, Q_m) of m = 0..3, tail m = 4.
// {} if the tables lack the delta structure.
static std::vector<double> direct_fragments5() {
  constexpr int P = 5;
  using S = DirShape5;
  std::vector<double> V, invD, RC, RS;
  build_tables_host(P, V, invD, &RC, &RS);
  auto rc = [&](int b, int m, int l) { return RC[((size_t)b * P + m) * P + l]; };
  auto rs = [&](int b, int m, int l) { return RS[((size_t)b * P + m) * P + l]; };
  // operator entry of (child b, element l) for output (m, P/Q):
  // P = RC_0 x_0 + RS_1 x_1, Q = RS_0 x_0 - RC_1 x_1
  auto opv = [&](int b, int l, int m, int pq) -> double {
    if (pq == 0) return b == 0 ? rc(0, m, l) : rs(1, m, l);
    return b == 0 ? rs(0, m, l) : -rc(1, m, l);
  };
  std::vector<double> fr(S::NFRAG, 0.0);
  for (int lane = 0; lane < 32; ++lane) {
    const int k = lane & 3, n = lane >> 2, c = lane & 3;
    const int b = k >> 1, l = 2 * (k & 1) + 1;
    fr[S::OFF_B + lane] = opv(b, l, n / 2, n % 2);
    fr[S::OFF_TAIL + lane] = opv(b, l, P - 1, 0);
    fr[S::OFF_TAIL + 32 + lane] = opv(b, l, P - 1, 1);
    const int m = c, l0 = 2 * m, l1 = 2 * m - (P - 1);
    const bool v0 = l0 <= P - 1, v1 = l1 >= 0;
    fr[S::OFF_DELTA + lane] = v0 ? opv(0, l0, m, 0) : 0.0;
    fr[S::OFF_DELTA + 32 + lane] = v0 ? opv(0, l0, m, 1) : 0.0;
    fr[S::OFF_DELTA + 64 + lane] = v1 ? opv(1, l1, m, 0) : 0.0;
    fr[S::OFF_DELTA + 96 + lane] = v1 ? opv(1, l1, m, 1) : 0.0;
    fr[S::OFF_DTAIL + lane] = c == 0 ? opv(1, P - 1, P - 1, 0) : 0.0;
    fr[S::OFF_DTAIL + 32 + lane] = c == 0 ? opv(1, P - 1, P - 1, 1) : 0.0;
  }
  // the split is exact only if every even-column entry outside the delta is 0
  for (int b = 0; b < 2; ++b)
    for (int l = 0; l < P; l += 2)
      for (int m = 0; m < P; ++m)
        if (2 * m != b * (P - 1) + l && (opv(b, l, m, 0) != 0.0 || opv(b, l, m, 1) != 0.0)) return {};
  return fr;
}

template <int P>
static const double* device_fragments(cudaError_t* err) {
  static std::mutex mu;
  static std::map<int, double*> cache;
  int dev = 0;
  if ((*err = cudaGetDevice(&dev)) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  std::vector<double> fr = UseSym<P>::v ? sym_fragments<P>() : direct_fragments5();
  if (fr.empty()) {  // the operator tables lack the symmetry / delta structure of the split
    *err = cudaErrorInvalidValue;
    return nullptr;
  }
  double* d = nullptr;
  if ((*err = cudaMalloc(&d, fr.size() * sizeof(double))) != cudaSuccess) return nullptr;
  if ((*err = cudaMemcpy(d, fr.data(), fr.size() * sizeof(double), cudaMemcpyHostToDevice)) != cudaSuccess)
    return nullptr;
  cache[dev] = d;
  return d;
}

// ------------------------------------------------------------------------
// launch configuration (tile of G groups per stage; tuned on B200)
// ------------------------------------------------------------------------
#ifndef SFT_F32_G29
#define SFT_F32_G29 8
#endif
#ifndef SFT_F32_NC29
#define SFT_F32_NC29 4
#endif
#ifndef SFT_F32_MINB29
#define SFT_F32_MINB29 4
#endif
#ifndef SFT_WS_G29
#define SFT_WS_G29 4
#endif
#ifndef SFT_WS_NC29
#define SFT_WS_NC29 4
#endif
#ifndef SFT_WS_NST29
#define SFT_WS_NST29 2
#endif
// G groups per tile, NC consumer warps, NST stages, MINB resident CTAs per SM
// (the register cap: MINB * (NC+1) warps share the 64K registers)
#ifndef SFT_WS_MINB29
#define SFT_WS_MINB29 4  // caps every variant (batch, two-level) at 96 registers: 4 CTAs per SM
#endif
template <int D, int P>
struct WsCfg;
#ifndef SFT_WS_G25
#define SFT_WS_G25 8
#endif
#ifndef SFT_WS_NC25
#define SFT_WS_NC25 4
#endif
#ifndef SFT_WS_NST25
#define SFT_WS_NST25 3
#endif
#ifndef SFT_WS_MINB25
#define SFT_WS_MINB25 3
#endif
#ifndef SFT_WS_G27
#define SFT_WS_G27 4
#endif
#ifndef SFT_WS_NC27
#define SFT_WS_NC27 4
#endif
#ifndef SFT_WS_NST27
#define SFT_WS_NST27 4
#endif
#ifndef SFT_WS_MINB27
#define SFT_WS_MINB27 4
#endif
// 2D p = 5 / 7 after the slot-major stage (translate ms, C0 | C2 geometry at p = 5:
// (16,4,3,2) 0.074 | 0.653, (8,4,3,3) 0.061 | 0.515, (4,4,3,4) 0.051 | 0.610; C1 | C2 geometry at
// p = 7: (8,4,3,3) 0.135 | 0.899, (4,4,4,4) 0.109 | 0.713, (2,4,3,4) 0.111 | 0.938)
template <> struct WsCfg<2, 5> {
  static constexpr int G = SFT_WS_G25, NC = SFT_WS_NC25, NST = SFT_WS_NST25, MINB = SFT_WS_MINB25;
};
template <> struct WsCfg<2, 7> {
  static constexpr int G = SFT_WS_G27, NC = SFT_WS_NC27, NST = SFT_WS_NST27, MINB = SFT_WS_MINB27;
};
template <> struct WsCfg<2, 9> {
  static constexpr int G = SFT_WS_G29, NC = SFT_WS_NC29, NST = SFT_WS_NST29, MINB = SFT_WS_MINB29;
};
// 3D configurations, overridable per field for sweeps (nvcc splits -D values at commas)
#ifndef SFT_WS_G35
#define SFT_WS_G35 1  // with the DMMA tail (80 registers): (1,4,2,5) C3 0.685 -> 0.672 ms vs (2,4,2,4)
#endif
#ifndef SFT_WS_NC35
#define SFT_WS_NC35 4
#endif
#ifndef SFT_WS_NST35
#define SFT_WS_NST35 2
#endif
#ifndef SFT_WS_MINB35
#define SFT_WS_MINB35 6  // 64 registers, no spills: C3 0.6226 -> 0.6206 ms
#endif
#ifndef SFT_WS_G37
#define SFT_WS_G37 1
#endif
#ifndef SFT_WS_NC37
#define SFT_WS_NC37 8
#endif
#ifndef SFT_WS_NST37
#define SFT_WS_NST37 2
#endif
#ifndef SFT_WS_MINB37
#define SFT_WS_MINB37 1
#endif
template <> struct WsCfg<3, 5> {
  static constexpr int G = SFT_WS_G35, NC = SFT_WS_NC35, NST = SFT_WS_NST35, MINB = SFT_WS_MINB35;
};
template <> struct WsCfg<3, 7> {
  static constexpr int G = SFT_WS_G37, NC = SFT_WS_NC37, NST = SFT_WS_NST37, MINB = SFT_WS_MINB37;
};
template <> struct WsCfg<3, 9> { static constexpr int G = 1, NC = 8, NST = 2, MINB = 1; };

#ifndef SFT_F2_WIDE
#define SFT_F2_WIDE 1  // two-level launches of <= one tile per SM: 12 consumer warps per CTA
#endif
static int sm_count() {
  static PerDevice<int> c;
  int v = 0;
  c.get(&v, [](int dev, int* r) { return cudaDeviceGetAttribute(r, cudaDevAttrMultiProcessorCount, dev); });
  return v > 0 ? v : 148;
}

// two-level launches (small plans, latency-bound): consumer warps per CTA and
// CTAs per SM (0 = the single-level configuration's)
#ifndef SFT_F2_NC
#define SFT_F2_NC 0
#endif
#ifndef SFT_F2_MINB
#define SFT_F2_MINB 0
#endif

// FP32 storage on the DMMA kernel (the FP32 variant): arrays are half the
// size, so twice the groups per stage at the same shared memory
template <int D, int P>
struct F32WsCfg;
template <> struct F32WsCfg<2, 5> { static constexpr int G = 16, NC = 4, NST = 3, MINB = 3; };
template <> struct F32WsCfg<2, 7> { static constexpr int G = 16, NC = 4, NST = 2, MINB = 3; };
template <> struct F32WsCfg<2, 9> { static constexpr int G = SFT_F32_G29, NC = SFT_F32_NC29, NST = 2, MINB = SFT_F32_MINB29; };
template <> struct F32WsCfg<3, 5> { static constexpr int G = 4, NC = 4, NST = 2, MINB = 3; };
template <> struct F32WsCfg<3, 7> { static constexpr int G = 2, NC = 8, NST = 2, MINB = 1; };
template <> struct F32WsCfg<3, 9> { static constexpr int G = 1, NC = 8, NST = 2, MINB = 1; };

static TransArgs make_args(const LevelDims& L, const double2* in, double2* out) {
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
  a.f2 = L.f2;
  a.cbK1 = L.cbK1;
  a.mK1 = L.mK1;
  a.cbX2 = L.cbX2;
  a.mX2 = L.mX2;
  if (L.f2) a.ngroups *= 4;  // virtual groups: the 2^d = 4 first-level groups of each super-group
  a.npeer = L.npeer;
  for (int q = 0; q < kMaxPeers; ++q) {
    a.peer[q] = L.peer[q];
    a.peer_off[q] = L.peer_off[q];
    a.peer_seg[q] = L.peer_seg[q];
  }
  a.peer_seg[kMaxPeers] = L.peer_seg[kMaxPeers];
  a.nrhs = L.nrhs;
  a.rs = L.rs;
  a.ctr = L.ctr;
  return a;
}

// Resident-CTA grid of a persistent kernel on the current device, with the
// kernel's dynamic shared-memory opt-in done once per device (a process may
// plan on several GPUs: nothing here is shared between devices).
// (cache: one per kernel instantiation -- the caller's static)
template <class K>
static cudaError_t persistent_grid(K kernel, int threads, size_t smem, int* grid, PerDevice<int>& cache) {
  return cache.get(grid, [&](int dev, int* out) {
    cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int nsm = 0, bps = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kernel, threads, smem);
    if (e != cudaSuccess) return e;
    if (bps < 1) return cudaErrorInvalidConfiguration;
    *out = nsm * bps;
    return cudaSuccess;
  });
}

// One persistent launch of k_translate_ws<D, P, G, NC, NST, MB, E, FUSED, BATCH, F2>
// NC: consumer warps of the producer design; the producer-less kernel (SFT_PL=1)
// runs NC + 1 consumers in the same (NC + 1) * 32 threads.  Measured slower
// (C2 translate 0.938 -> 1.042 ms, C3 0.714 -> 0.778, C4 32.0 -> 35.4): the
// refill work lands on a consumer, and one more warp per pass barrier gets
// fewer super-tiles each; off.
#ifndef SFT_PL
#define SFT_PL 0
#endif
template <int D, int P, int G, int NC, int NST, int MB, typename E, bool FUSED, bool BATCH, bool F2>
static cudaError_t launch_ws(const sft_plan_s* Pl, const TransArgs& a, const LevelDims& L, int64_t work) {
  constexpr int PS = StrideT<E, Pow<P, D>::v>::v;
  const size_t smem = ((size_t)NST * (1 << D) * (G * PS + SlotPad<D, P, PS>::v) + PS) * sizeof(E);  // ring + zero slot
  constexpr bool PLK = SFT_PL != 0;
  constexpr int NCK = PLK ? NC + 1 : NC;
  auto kern = k_translate_ws<D, P, G, NCK, NST, MB, E, FUSED, BATCH, F2, PLK>;
  static PerDevice<int> grid_cache;  // this instantiation's grid and smem opt-in, per device
  int grid_max = 0;
  cudaError_t e = persistent_grid(kern, (NC + 1) * 32, smem, &grid_max, grid_cache);
  if (e != cudaSuccess) return e;
  const double* frag = device_fragments<P>(&e);
  if (!frag) return e;
  const int64_t ntiles = (a.ngroups + G - 1) / G;
  // dynamic tile scheduling pays with many items per CTA (C2 translate 0.936 ->
  // 0.892 ms, C3 0.671 -> 0.632, C4 31.8 -> 30.4); with a few per CTA the
  // counter's latency is exposed (C1 0.072 -> 0.076): grid-stride there
  TransArgs ad = a;
  if (work <= 4 * (int64_t)grid_max) ad.ctr = nullptr;
  launch_pdl(kern, (unsigned)std::min<int64_t>(work, grid_max), (NC + 1) * 32, smem, Pl->stream, ad, frag, L.sched,
             ntiles);
  count_launch();
  return cudaGetLastError();
}

template <int D, int P>
static cudaError_t launch_translate_t(const sft_plan_s* Pl, const LevelDims& L, const void* in, void* out) {
  TransArgs a = make_args(L, (const double2*)in, (double2*)out);
  if (a.ngroups <= 0) return cudaSuccess;
  if (!L.sched) return cudaErrorInvalidValue;
  if (a.nrhs < 1 || (a.nrhs > 1 && a.npeer > 0)) return cudaErrorInvalidValue;
  if (a.f2 && (Pl->prec != 0 || a.npeer > 0)) return cudaErrorInvalidValue;  // two-level: FP64 only
  if (Pl->prec == 1) {
    // FP32 storage, FP64 arithmetic on the tensor cores (same kernel as FP64)
    using C = F32WsCfg<D, P>;
    const int64_t work = (a.ngroups + C::G - 1) / C::G * a.nrhs;
    if (a.nrhs > 1) return launch_ws<D, P, C::G, C::NC, C::NST, C::MINB, float2, false, true, false>(Pl, a, L, work);
    return launch_ws<D, P, C::G, C::NC, C::NST, C::MINB, float2, false, false, false>(Pl, a, L, work);
  }
  using C = WsCfg<D, P>;
  const int64_t work = (a.ngroups + C::G - 1) / C::G * a.nrhs;
  if (a.npeer > 0) return launch_ws<D, P, C::G, C::NC, C::NST, C::MINB, double2, true, false, false>(Pl, a, L, work);
  if (a.f2) {
    // two-level launch (2D, G = 4k; the unskewed pipeline, so at most 2 stages
    // even where single-level launches of that p use the skewed one)
    if constexpr (D == 2 && C::G % 4 == 0) {
      constexpr int NST2 = C::NST < 3 ? C::NST : 2;
      constexpr int NC2 = SFT_F2_NC > 0 ? SFT_F2_NC : C::NC, MINB2 = SFT_F2_MINB > 0 ? SFT_F2_MINB : C::MINB;
      if (a.nrhs > 1) return launch_ws<D, P, C::G, NC2, NST2, MINB2, double2, false, true, true>(Pl, a, L, work);
      // at most one tile per SM (C0's levels): the launch is one tile's latency
      // chain, so a CTA of 12 consumer warps (fewer super-tiles per warp per
      // pass) finishes sooner -- C0 translate 0.031 -> 0.027 ms; with more
      // tiles than SMs the narrower, more numerous CTAs win (C1)
      if (SFT_F2_WIDE && work <= sm_count())
        return launch_ws<D, P, C::G, 12, NST2, 1, double2, false, false, true>(Pl, a, L, work);
      return launch_ws<D, P, C::G, NC2, NST2, MINB2, double2, false, false, true>(Pl, a, L, work);
    }
    return cudaErrorInvalidValue;
  }
  if (a.nrhs > 1) return launch_ws<D, P, C::G, C::NC, C::NST, C::MINB, double2, false, true, false>(Pl, a, L, work);
  return launch_ws<D, P, C::G, C::NC, C::NST, C::MINB, double2, false, false, false>(Pl, a, L, work);
}

template <int D, int P, int G>
static size_t schedule_bytes_g(const LevelDims& L) {
  const int64_t ng = (L.b_hi - L.b_lo) * (L.ap_hi - L.ap_lo) * (L.f2 ? 4 : 1);  // f2: virtual groups
  if (ng <= 0) return 0;
  return (size_t)((ng + G - 1) / G) * Sched<D, P, G>::BLK * (L.f2 ? 2 : 1);  // f2: one block per level
}

template <int D, int P>
static size_t schedule_bytes_t(const sft_plan_s* Pl, const LevelDims& L) {
  if (Pl->prec == 1) return schedule_bytes_g<D, P, F32WsCfg<D, P>::G>(L);
  return schedule_bytes_g<D, P, WsCfg<D, P>::G>(L);
}

template <int D, int P, int G, int PS>
static cudaError_t launch_schedule_g(const sft_plan_s* Pl, const LevelDims* L, int nlev, unsigned char* const* dst,
                                     cudaStream_t st) {
  // two passes over the levels: single-level schedules, then two-level ones
  for (int f2 = 0; f2 < 2; ++f2) {
    std::vector<int> idx;
    for (int i = 0; i < nlev; ++i)
      if ((L[i].f2 != 0) == (f2 != 0)) idx.push_back(i);
    for (size_t c0 = 0; c0 < idx.size(); c0 += kSchedChunk) {
      SchedLevels S;
      int64_t t0 = 0;
      S.nlev = 0;
      for (size_t q = c0; q < idx.size() && q < c0 + kSchedChunk; ++q) {
        const int i = idx[q];
        TransArgs a = make_args(L[i], nullptr, nullptr);
        if (a.ngroups <= 0) continue;
        S.a[S.nlev] = a;
        S.dst[S.nlev] = dst[i];
        S.ctr[S.nlev] = L[i].ctr;
        S.tile0[S.nlev] = t0;
        t0 += (a.ngroups + G - 1) / G;
        ++S.nlev;
      }
      S.tile0[S.nlev] = t0;
      if (S.nlev == 0) continue;
      const int64_t nwarps = (t0 + 32 / G - 1) / (32 / G);
      if (f2)
        k_schedule<D, P, G, PS, true><<<(unsigned)((nwarps + 3) / 4), 128, 0, st>>>(S);
      else
        k_schedule<D, P, G, PS><<<(unsigned)((nwarps + 3) / 4), 128, 0, st>>>(S);
      count_launch();
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
  }
  return cudaSuccess;
}

template <int D, int P>
static cudaError_t launch_schedule_t(const sft_plan_s* Pl, const LevelDims* L, int nlev, unsigned char* const* dst,
                                     cudaStream_t st) {
  if (Pl->prec == 1)
    return launch_schedule_g<D, P, F32WsCfg<D, P>::G, StrideT<float2, Pow<P, D>::v>::v>(Pl, L, nlev, dst, st);
  return launch_schedule_g<D, P, WsCfg<D, P>::G, StrideT<double2, Pow<P, D>::v>::v>(Pl, L, nlev, dst, st);
}

template <int D, int P>
static cudaError_t check_schedule_t(const sft_plan_s* Pl, const LevelDims& L, const unsigned char* sched,
                                   int64_t in_pairs, int64_t out_pairs, int* err) {
  if (Pl->prec != 0 || L.f2) return cudaSuccess;  // (single-level layout only)
  constexpr int G = WsCfg<D, P>::G;
  TransArgs a = make_args(L, nullptr, nullptr);
  if (a.ngroups <= 0) return cudaSuccess;
  const int64_t ntiles = (a.ngroups + G - 1) / G;
  k_check_schedule<D, P, G><<<(unsigned)((ntiles + 127) / 128), 128, 0, Pl->stream>>>(a, sched, ntiles, in_pairs,
                                                                                       out_pairs, err);
  return cudaGetLastError();
}

cudaError_t check_schedule(const sft_plan_s* Pl, const LevelDims& L, const unsigned char* sched, int64_t in_pairs,
                           int64_t out_pairs, int* err) {
  SFT_DISPATCH(Pl->d, Pl->p, return (check_schedule_t<D, P>(Pl, L, sched, in_pairs, out_pairs, err)));
  return cudaSuccess;
}

static cudaError_t schedule_bytes_d(const sft_plan_s* Pl, const LevelDims& L, size_t* r) {
  SFT_DISPATCH(Pl->d, Pl->p, (*r = schedule_bytes_t<D, P>(Pl, L)));
  return cudaSuccess;
}

size_t schedule_bytes(const sft_plan_s* Pl, const LevelDims& L) {
  size_t r = 0;
  schedule_bytes_d(Pl, L, &r);
  return r;
}

cudaError_t launch_schedule(const sft_plan_s* Pl, const LevelDims* L, int nlev, unsigned char* const* dst,
                            cudaStream_t st) {
  SFT_DISPATCH(Pl->d, Pl->p, return (launch_schedule_t<D, P>(Pl, L, nlev, dst, st)));
  return cudaSuccess;
}

// FP64 flops one warp executes per 8-fiber super-tile (DMMA m8n8k4: 512 flops
// incl. padding; DADD / DMUL: 32, DFMA: 64 per warp instruction), counted
// from sym_math / direct_math (NSUB = 1 code; NSUB only interleaves):
//   symmetric p = 7: 4 DMMA, 16 DADD, 8 DMUL, 8 DFMA
//   symmetric p = 9: 8 DMMA, 24 DADD, 12 DMUL, 8 DFMA (centre tile; SFT_CENTRE_DMMA=0:
//                    4 DMMA, 27 DADD, 12 DMUL, 12 DFMA with the centre tail)
//   direct    p = 5: 2 DMMA, 11 DADD, 8 DMUL, 8 DFMA (tail)
static double flops_per_supertile(int p) {
  if (p == 5) return 2 * 512 + 11 * 32 + 8 * 32 + 8 * 64;
  if (p == 7) return 4 * 512 + 16 * 32 + 8 * 32 + 8 * 64;
  if (SFT_CENTRE_DMMA) return 8 * 512 + 24 * 32 + 12 * 32 + 8 * 64;
  return 4 * 512 + 27 * 32 + 12 * 32 + 12 * 64;
}

template <int D, int P, int G>
static void schedule_work_g(const unsigned char* h, size_t bytes, int nb, double* out) {
  using SC = Sched<D, P, G>;
  constexpr int PF = Pow<P, D>::v / P;
  const size_t blk = (size_t)SC::BLK;
  double st = 0, tasks = 0;
  for (size_t o = 0; o + blk <= bytes; o += blk) {
    const int* cnt = reinterpret_cast<const int*>(h + o);
    for (int l = 0; l < SC::NCNT; ++l) {  // (3D: every sub-list is its own super-tile loop)
      const int nt = cnt[3 * l] + cnt[3 * l + 1] + cnt[3 * l + 2];
      tasks += nt;
      st += (nt * PF + 7) / 8;
    }
  }
  (void)nb;
  out[0] += st;
  out[1] += tasks;
  out[2] += st * flops_per_supertile(P);
}

// Work of one translation launch from its tile schedule (host copy): out[0]
// super-tiles, out[1] fiber tasks, out[2] executed FP64 flops (accumulated).
void schedule_work(const sft_plan_s* Pl, const unsigned char* h, size_t bytes, double* out) {
  if (Pl->prec == 1) {
    switch (Pl->d * 10 + Pl->p) {
      case 25: return schedule_work_g<2, 5, F32WsCfg<2, 5>::G>(h, bytes, 1, out);
      case 27: return schedule_work_g<2, 7, F32WsCfg<2, 7>::G>(h, bytes, 1, out);
      case 29: return schedule_work_g<2, 9, F32WsCfg<2, 9>::G>(h, bytes, 1, out);
      case 35: return schedule_work_g<3, 5, F32WsCfg<3, 5>::G>(h, bytes, 1, out);
      case 37: return schedule_work_g<3, 7, F32WsCfg<3, 7>::G>(h, bytes, 1, out);
      case 39: return schedule_work_g<3, 9, F32WsCfg<3, 9>::G>(h, bytes, 1, out);
    }
    return;
  }
  switch (Pl->d * 10 + Pl->p) {
    case 25: return schedule_work_g<2, 5, WsCfg<2, 5>::G>(h, bytes, 1, out);
    case 27: return schedule_work_g<2, 7, WsCfg<2, 7>::G>(h, bytes, 1, out);
    case 29: return schedule_work_g<2, 9, WsCfg<2, 9>::G>(h, bytes, 1, out);
    case 35: return schedule_work_g<3, 5, WsCfg<3, 5>::G>(h, bytes, 1, out);
    case 37: return schedule_work_g<3, 7, WsCfg<3, 7>::G>(h, bytes, 1, out);
    case 39: return schedule_work_g<3, 9, WsCfg<3, 9>::G>(h, bytes, 1, out);
  }
}

bool two_level_supported(const sft_plan_s* Pl) {
  if (Pl->prec != 0 || Pl->sharded) return false;
  const char* e = getenv("SFT_F2");
  if (e && e[0] == '0') return false;
  if (Pl->d != 2) return false;
  switch (Pl->p) {
    case 5: return WsCfg<2, 5>::G % 4 == 0;
    case 7: return WsCfg<2, 7>::G % 4 == 0;
    case 9: return WsCfg<2, 9>::G % 4 == 0;
  }
  return false;
}

cudaError_t launch_translate(const sft_plan_s* Pl, const LevelDims& L, const void* in, void* out) {
  SFT_DISPATCH(Pl->d, Pl->p, return (launch_translate_t<D, P>(Pl, L, in, out)));
  return cudaSuccess;
}

}  // namespace sft

#ifdef SFT_INSTR
extern "C" int sft_instr_set(void* dev_buf) {
  return cudaMemcpyToSymbol(sft::g_instr, &dev_buf, sizeof(void*)) == cudaSuccess ? 0 : 4;
}
#endif
