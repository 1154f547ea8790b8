/*
 * sft.h -- C ABI of the B200 butterfly sparse Fourier transform (libsft.so).
 *
 * Computes u_i = sum_j exp(2*pi*i * x_i . k_j / N) f_j          (eq. sfft)
 * with Ying's butterfly algorithm (§2.2):
 *   sft_plan   -- step 1, quadtrees/octrees T_X, T_K of non-empty boxes with
 *                 unit-width leaves, built on the GPU;
 *   sft_apply  -- step 2 leaf charges, step 3 per-level
 *                 translations (fig. 1), step 4 final
 *                 evaluation; all in hand-written sm_100a kernels;
 *   sft_destroy.
 *
 * Conventions:
 *   - dim in {2,3}; N = 2^L with 2 <= N <= 2^20; p in {5,7,9} (grid points per
 *     axis).  Points must lie in [0,N]^dim; a point with
 *     coordinate y belongs to leaf floor(y) (N-1 when y == N).
 *   - Layouts: x [nx][dim], k [nk][dim] float64 row-major (torch.float64 [n,dim]);
 *     f [nk], u [nx] complex128 with (re,im) interleaved (torch.complex128).
 *   - Pointers may be host or device memory (detected with
 *     cudaPointerGetAttributes).  Host buffers are staged through plan-owned
 *     device memory inside the call (this is the "e2e" path of bench.py).
 *   - Ownership: the caller owns x, k, f, u.  sft_plan copies what it needs
 *     (sorted coordinates), so x and k may be freed after it returns.  The plan
 *     owns trees, operator tables and the two live level buffers
 *     until sft_destroy.
 *   - Streams: all device work of a plan is ordered on opts.stream (a
 *     cudaStream_t; NULL = legacy default stream).  sft_plan synchronises that
 *     stream once (to size the level buffers).  sft_apply does not synchronise
 *     unless f or u is a host pointer.
 *   - Errors: every call returns an SFT_* status; nothing throws across the ABI;
 *     a failed sft_plan leaves *out untouched.  sft_last_error() gives a
 *     thread-local message for the last failure.
 *   - Semantics: linear in f; f == 0 gives u == 0 exactly; deterministic (no
 *     floating-point atomics; identical bits run to run and for any world size).
 *     One plan must not be used by two concurrent sft_apply calls.
 */
#ifndef SFT_H_
#define SFT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SFT_OK = 0,
  SFT_E_ARG = 1,     /* bad dim/N/p/count/pointer/option */
  SFT_E_DOMAIN = 2,  /* a coordinate is non-finite or outside [0,N] */
  SFT_E_NOMEM = 3,   /* device or host allocation failed */
  SFT_E_CUDA = 4,    /* CUDA runtime error (message in sft_last_error) */
  SFT_E_STATE = 5,   /* call not valid for this plan (e.g. phase order, world size) */
  SFT_E_NCCL = 6,    /* NCCL unavailable or a collective failed (message in sft_last_error) */
};

typedef struct sft_plan_s* sft_plan_t;

typedef struct {
  int precision;      /* 0 = FP64 (default); 1 = FP32 storage of the level charges
                       *     (operators, leaf/final arithmetic and tensor-core
                       *     accumulation stay FP64; ~1e-6 relative error; world == 1 only) */
  void* stream;       /* cudaStream_t for all device work; NULL = default stream */
  int rank;           /* this rank's index, 0 <= rank < world */
  int world;          /* number of ranks sharing the transform; 1 = single GPU */
  int exchange_level; /* world > 1: level m of the charge exchange; -1 = choose */
  int split_k;        /* world > 1: T_K subtree level s_K; -1 = choose */
  int split_x;        /* world > 1: T_X subtree level s_X; -1 = choose */
  int adjoint;        /* 1: the plan applies the adjoint transform
                       *    v_j = sum_i exp(-2*pi*i x_i . k_j / N) g_i   (g on the x points,
                       *    v on the k points; eq. sfft conjugate-transposed) -- the same
                       *    butterfly with the roles of the point sets swapped and the
                       *    charges / potentials conjugated; sft_apply then takes g [nx]
                       *    and writes v [nk].  0 = forward (default).  world == 1 only. */
  const void* nccl_id;  /* world > 1: a 128-byte ncclUniqueId (from sft_nccl_unique_id on one
                         * rank, broadcast to all ranks by the caller, e.g. torch.distributed).
                         * With it, sft_plan joins / reuses the NCCL communicator of that id
                         * (ncclCommInitRank on the first plan of a rank with this id: every
                         * rank must plan concurrently) and sft_apply runs the whole sharded
                         * transform, exchange and u all-gather included.  NULL (default):
                         * the caller drives the phase calls and the collective itself.
                         * world == 1 with nccl_id and exchange_level >= 0 runs the sharded
                         * path on a single rank (self send/recv; a test of the machinery). */
} sft_opts;

/* Fill *o with defaults: FP64, NULL stream, rank 0, world 1, automatic levels, forward,
 * no NCCL id. */
void sft_default_opts(sft_opts* o);

/* Step 1: build T_X from targets x and T_K from sources k.
 * x: [nx][dim] float64, k: [nk][dim] float64 (host or device), nx, nk >= 1.
 * Returns SFT_E_ARG for bad dim/N/p/counts/NULL pointers, SFT_E_DOMAIN for a
 * coordinate outside [0,N] or non-finite. */
int sft_plan(int dim, int64_t N, int p, const double* x, int64_t nx, const double* k, int64_t nk,
             const sft_opts* opts, sft_plan_t* out);

/* Steps 2-4: u = butterfly(f).  f: [nk] complex128, u: [nx]
 * complex128, host or device.  A host f may be modified as soon as the call
 * returns (the call waits for its staging copy); a host u is complete on return.
 * Sharded plans (world > 1) need opts.nccl_id at plan time: every rank passes
 * the full f and gets the full u -- phase 1 over its T_K subtrees, the level-m
 * exchange as grouped ncclSend/ncclRecv, phase 2 over its T_X subtrees, an
 * ncclAllGather of the potentials and a scatter to user order, all on the plan
 * stream; bitwise equal to the world == 1 result.
 * SFT_E_STATE for a sharded plan without an NCCL id (use the phase calls);
 * SFT_E_NCCL if a collective fails. */
int sft_apply(sft_plan_t plan, const void* f, void* u);

/* Multi-RHS apply: u_r = butterfly(f_r) for nrhs
 * charge vectors through one plan, r = 0..nrhs-1.  f_r at f + r*ldf and u_r at
 * u + r*ldu (complex128 elements, ldf >= nk, ldu >= nx); f and u host or device.
 * Same arithmetic per vector as sft_apply (bitwise identical results), but one
 * launch per step for all vectors: the leaf weights and final-step powers are
 * computed once per point and the tile schedules once per tile for the whole
 * batch.  Needs nrhs x the plan's level-buffer bytes of extra device memory
 * (allocated on the first call and kept; SFT_E_NOMEM if it does not fit).
 * 1 <= nrhs <= 4096; world == 1 plans only (SFT_E_STATE otherwise). */
int sft_apply_batch(sft_plan_t plan, int nrhs, const void* f, int64_t ldf, void* u, int64_t ldu);

/* Far-field adapter (eq. far): a plan whose sft_apply computes
 *   u_inf(xhat_i) = sum_j exp(-i kappa xhat_i . y_j) F_j
 * (F_j = f(y_j) ds_j, the quadrature-weighted density on the scatterer
 * boundary; kappa = the wave number, written N in eq. far).
 *   xhat: [nx][dim] unit directions, y: [ny][dim] points in [0,1]^dim
 *   (float64 row-major, host or device; the caller rescales the scatterer
 *   into the unit box).  kappa in (0, pi 2^20].
 * The SFT size is N = the smallest power of two >= max(2, kappa/pi); the
 * points become x = N/2 - kappa xhat/(2 pi) and k = N y (a kernel), so that
 * 2 pi x.k/N = pi sum_a k_a - kappa xhat.y: "after we rescale xhat and y by a
 * factor of N, (far) takes the form of (sfft)".  The leftover
 * phase e^{i pi sum_a k_a} is folded into the leaf kernel (a sign per leaf
 * box).  opts->adjoint = 1 gives the adjoint v_j = sum_i exp(+i kappa
 * xhat_i . y_j) g_i (g on the directions, v on the scatterer points; the
 * phase then goes into the final kernel).  sft_apply / sft_apply_batch /
 * sft_destroy as for any plan; world == 1 only.  Errors as sft_plan, plus
 * SFT_E_ARG for a bad kappa; SFT_E_DOMAIN if a y is outside [0,1]^dim or a
 * |xhat_a| > 1. */
int sft_farfield_plan(int dim, double kappa, int p, const double* xhat, int64_t nx, const double* y, int64_t ny,
                      const sft_opts* opts, sft_plan_t* out);

/* NULL is a no-op. */
int sft_destroy(sft_plan_t plan);

const char* sft_strerror(int status);
const char* sft_last_error(void);

/* Plan statistics (host memory, caller-allocated).
 *   counts_x, counts_k: [L+1] non-empty boxes per level of T_X / T_K (or NULL)
 *   pairs: [L+1] pairs(t) = |T_K level t| * |T_X level L-t| (or NULL)
 *   info[0..7]: L, p^dim, nx, nk, level-buffer bytes, plan ms (device),
 *               groups total, translation algorithmic bytes per apply. */
int sft_plan_stats(sft_plan_t plan, int64_t* counts_x, int64_t* counts_k, int64_t* pairs, double* info);

/* Work model of one sft_apply's translation step (host, caller-allocated [6];
 * synchronises the plan stream once; diagnostics for the roofline):
 *   w[0] algorithmic bytes: every pair array written once at its level and
 *        read once at the next (the level-synchronous schedule)
 *   w[1] FP64 flops the translation kernels execute (DMMA m8n8k4 tiles
 *        counted whole, padding included, plus the DADD/DMUL/DFMA of the
 *        delta columns, sum/difference and tail), from the tile schedules
 *   w[2] 8-fiber super-tiles, w[3] fiber tasks, w[4] groups (A', B),
 *   w[5] pairs (A, B) over all levels. */
int sft_plan_work(sft_plan_t plan, double* w);

/* Translation launches of sft_apply (host, caller-allocated [L] arrays or NULL):
 * *n launches in order; out_level[i] = the level t the launch writes;
 * two_level[i] = 1 if it is a two-level (radix-4) launch computing levels t+1
 * and t from level t+2 in one pass over super-groups (A'', B) without storing
 * level t+1 (SURVEY.md §8(f) item 2 "cross-level fusion"; 2D FP64 single-GPU
 * plans; SFT_F2=0 disables), else a single-level launch. */
int sft_translation_launches(sft_plan_t plan, int* n, int* out_level, int* two_level);

/* Device time (ms, CUDA events on the plan stream) of the kernels of the last
 * sft_apply when timing was enabled with sft_set_timing(plan, mode):
 *   t_ms[0] leaf kernel, t_ms[1] sum of translation kernels, t_ms[2] final
 *   kernel, t_ms[3] whole apply; per_level_ms [L] translation level t=0..L-1
 *   (or NULL; a two-level launch is booked on its output level t, level t+1
 *   then reads 0).  mode 1: an event after every launch (per-level times; the
 *   events cut the programmatic-dependent-launch overlap between levels);
 *   mode 2: events only around the leaf kernel, the whole translation chain
 *   and the final kernel (t_ms[1] = the chain, per_level_ms all 0).  mode 0:
 *   off; other modes: SFT_E_ARG.  Multi-rank plans: after sft_apply_phase2,
 *   t_ms[1] is this rank's translation time of both phases (the other entries
 *   are not set). */
int sft_set_timing(sft_plan_t plan, int enable);
int sft_last_timing(sft_plan_t plan, double* t_ms, double* per_level_ms);

/* NCCL id for opts.nccl_id (ncclGetUniqueId; libnccl.so.2 is dlopen'ed: the
 * NCCL already loaded in the process, e.g. torch's, is used).  id128: 128
 * bytes.  SFT_E_NCCL if NCCL cannot be loaded. */
int sft_nccl_unique_id(void* id128);
/* Destroy this process's communicators of that id (plans using it must be
 * destroyed first).  Unknown ids are a no-op. */
int sft_nccl_release(const void* id128);

/* ---- multi-GPU (world > 1), SURVEY.md §8(e) ----------------------------
 * Phase 1 (levels t = L..m) over this rank's T_K subtrees at level s_K,
 * one all-to-all of the level-m charges, phase 2 (t = m-1..0 and step 4) over
 * this rank's T_X subtrees at level s_X.  With opts.nccl_id sft_apply does all
 * of it; the phase calls below let the caller drive the steps and the
 * collective itself (torch.distributed, the fused exchange, tests).
 *
 * sft_exchange_counts: send_counts/recv_counts [world] in complex128 elements
 *   (contiguous per-peer segments in rank order).
 * sft_apply_phase1(plan, f, sendbuf): f [nk] (all sources); sendbuf device,
 *   >= sum(send_counts) complex128.
 * sft_apply_phase2(plan, recvbuf, u): recvbuf device with the peers' segments
 *   concatenated in rank order; u [nx] is fully overwritten: this rank's
 *   targets get their values, all others 0 (sum-reduce across ranks to
 *   assemble; every entry has exactly one non-zero contributor). */
int sft_exchange_counts(sft_plan_t plan, int64_t* send_counts, int64_t* recv_counts);
int sft_apply_phase1(sft_plan_t plan, const void* f, void* sendbuf);
int sft_apply_phase2(sft_plan_t plan, const void* recvbuf, void* u);

/* Fused exchange (compute + collective in one kernel over NVLink peer memory):
 * sft_set_peer_buffers(plan, recv): recv[world] = every rank's receive buffer
 *   (device pointers valid in this process: own buffer for this rank, peers'
 *   buffers opened with sft_ipc_open).  Afterwards sft_apply_phase1 writes the
 *   level-m charges straight into the receivers' buffers from the epilogue of
 *   the exchange level's translation kernel (sendbuf may be NULL) -- the
 *   caller only needs a stream-ordered barrier across ranks before
 *   sft_apply_phase2.  recv == NULL switches back to the send buffer.
 * sft_peer_offsets(plan, off[world]): element offset of this rank's segment in
 *   each receiver's buffer.
 * Device memory that can be shared across processes (cudaMalloc, not the
 * stream-ordered pool): sft_device_alloc / sft_device_free; CUDA IPC:
 * sft_ipc_handle(ptr, handle[64 bytes]) / sft_ipc_open(handle, &ptr) /
 * sft_ipc_close(ptr).  world <= 8. */
int sft_set_peer_buffers(sft_plan_t plan, void* const* recv);
int sft_peer_offsets(sft_plan_t plan, int64_t* off);
int sft_device_alloc(int64_t bytes, void** out);
int sft_device_free(void* p);
int sft_ipc_handle(void* p, void* handle64);
int sft_ipc_open(const void* handle64, void** out);
int sft_ipc_close(void* p);

/* Partition actually used by a world > 1 plan (host, caller-allocated):
 * part[0..2] = s_K, s_X, m; then for every rank r: part[3+4r .. 3+4r+3] =
 * [first, last) T_K box range at level s_K and [first, last) T_X box range at
 * level s_X owned by r (Morton order, contiguous). */
int sft_partition_info(sft_plan_t plan, int64_t* part);

/* Host-only partitioner (no GPU needed; sft_plan calls the same routine).
 * counts_x/counts_k: [L+1] non-empty boxes per level; parent_x/parent_k: [L+1]
 * pointers, parent_*[l] = [counts[l]] int32 parent index (level l-1) of each
 * box at level l (entry 0 unused).  force_*: -1 = choose, else use the value.
 * Chooses (s_K, s_X, m) and contiguous subtree ranges minimising
 *   max_r phase-1 pairs + max_r phase-2 pairs + 4 * max_r exchanged pairs
 * (pairs ~ p^d*16 bytes of HBM traffic each; one exchanged pair over NVLink
 * costs ~4 pairs of HBM time).  out: [3 + 4*world] laid out as in
 * sft_partition_info; out_cost (may be NULL): [3] the three max terms. */
int sft_choose_partition(int L, int world, const int64_t* counts_x, const int64_t* counts_k,
                         const int32_t* const* parent_x, const int32_t* const* parent_k, int force_sk,
                         int force_sx, int force_m, int64_t* out, int64_t* out_cost);

/* Diagnostics: the tile schedule of translation level t (built by sft_plan
 * for the translation kernel: per tile of groups, task counts, child-array
 * sources and task records; layout in translate.cu).  *bytes = its size;
 * if dst (host) is non-NULL the schedule is copied there (synchronises the
 * plan stream). */
int sft_schedule_bytes(sft_plan_t plan, int t, int64_t* bytes, void* dst);

/* Number of kernels launched by this library since load (its own kernels;
 * the CUB radix-sort/scan kernels used by the tree build are not counted). */
int sft_launch_count(int64_t* out);

/* Diagnostics (host only, no GPU): the constant operator tables for grid
 * size p (3 <= p <= 15), built in long double from the Lagrange /
 * sine-product closed forms:
 *   V    [2][2][p][p] complex128 interleaved: the child->parent operator
 *        V[alpha][beta][m][l'] in box-relative charges g (= M^{-1} E);
 *   invD [p] leaf-weight normalisers 1/prod_{q!=m} sin(pi (m-q)/(p-1)^2);
 *   RC, RS [2][p][p] float64: the real operands the translation kernel keeps
 *        in the constant bank (T = c (RC + i s_alpha RS) in the h-representation).
 * Any pointer may be NULL. */
int sft_operator_tables(int p, double* V, double* invD, double* RC, double* RS);

#ifdef __cplusplus
}
#endif

#endif /* SFT_H_ */
