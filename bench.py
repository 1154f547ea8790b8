#!/usr/bin/env python
"""Benchmark of the B200 butterfly sparse Fourier transform (arXiv 0801.1524).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl ours|reference]

One step = one pass of the whole hot path (plus
S5 for N > 1) on the workload: sft_plan (GPU tree build, step 1 P:293-295)
followed by sft_apply (leaf, per-level translations, final), with
x, k, f resident in HBM.  Metric (BASELINE.json:2): Mpoints/s = P / step time
with P = max(n_x, n_k) (the paper's P); apply-only ms is
reported beside it.  L2 is flushed (256 MiB memset) before every timed step;
each step is timed with CUDA events on the plan stream, max over ranks.

N > 1: one process per GPU under torchrun; the transform is sharded
(phase 1 over T_K subtrees, NCCL all-to-all of level-m charges, phase 2 over
T_X subtrees) -- strong scaling of one transform.

--impl reference: the oracle (oracle/, long double CPU) on the box's host
cores, rank 0 only (the other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

CONFIG_DESC = {
    "C0": "2D N=64 p=5, X=K=circle r=0.4, 4 pts/unit length, f ~ CN(0,1) seed 0 (BASELINE.json:7)",
    "C1": "2D N=1024 p=7, X circle r=0.4, K ellipse (0.35,0.25), 4 pts/unit length, seed 1 (BASELINE.json:8)",
    "C2": "2D N=16384 p=9, X circle r=0.4, K ellipse (0.35,0.25), 4 pts/unit length, seed 2 (BASELINE.json:9)",
    "C3": "3D N=128 p=5, X sphere r=0.4, K ellipsoid (0.4,0.3,0.25), lat-long 2 pts/unit length, seed 3 (BASELINE.json:10)",
    "C4": "3D N=512 p=7, X sphere r=0.4, K ellipsoid (0.4,0.3,0.25), lat-long 2 pts/unit length, seed 4 (BASELINE.json:11)",
}


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peak():
    """FP64 tensor-core (DMMA m8n8k4) peak measured on this pool's B200 with
    scripts/fp64_peak.cu (profiles/r1_fp64_peak.json; MEASURED_PEAKS.json has
    no FP64 entry): 36.85 TF/s at 1.96 GHz.  DFMA reaches 34-39 TF/s on the same
    datapath (mixed DMMA + DFMA: 32.4 TF/s total)."""
    path = os.path.join(ROOT, "profiles", "r1_fp64_peak.json")
    try:
        for line in open(path):
            d = json.loads(line)
            if d.get("test") == "dmma_m8n8k4":
                return float(d["tflops"]), "measured (profiles/r1_fp64_peak.json, DMMA m8n8k4)"
    except OSError:
        pass
    return 37.2, "nominal (148 SMs x 64 FP64 FMA/clk x 2 x 1.965 GHz)"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    """SM clock and clock-event (throttle) reasons sampled during the timed
    region: NVML polled every ~1 ms from a thread (the timed regions are tens
    of ms, too short for `nvidia-smi -lms`), nvidia-smi as the fallback."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = int(gpu_index)
        self.proc = None
        self.lines = []
        self.t = None
        self.nv = None
        self.samples = []  # (sm_mhz, reasons bitmask)
        self.stop_flag = threading.Event()

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            idx = self.gpu
            if vis:
                try:
                    idx = int(vis.split(",")[self.gpu])
                except ValueError:
                    idx = self.gpu
            self.nv = (pynvml, pynvml.nvmlDeviceGetHandleByIndex(idx))
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.nv[1], pynvml.NVML_CLOCK_SM)
            self.sample_once()
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def sample_once(self):
        nv, h = self.nv
        self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                             nv.nvmlDeviceGetCurrentClocksEventReasons(h)))

    def _poll(self):
        while not self.stop_flag.is_set():
            try:
                self.sample_once()
            except Exception:
                break
            time.sleep(0.001)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.nv is not None:
            self.stop_flag.set()
            self.t.join(timeout=5)
            try:
                self.sample_once()
            except Exception:
                pass
            nv = self.nv[0]
            names = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                     "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                     "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                     "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
            reasons = sorted({n for _, r in self.samples for n, bit in names.items() if r & bit})
            sm = [float(c) for c, _ in self.samples]
            busy = [v for v in sm if v > 0.5 * self.max_mhz] or sm
            return {"sm_mhz": float(np.median(busy)) if busy else None, "sm_max_mhz": float(self.max_mhz),
                    "samples": len(sm), "reasons": reasons, "source": "nvml"}
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=5)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx = float(parts[2])
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        busy = [v for v in sm if v > 0.5 * (mx or 1)] or sm
        return {"sm_mhz": float(np.median(busy)) if busy else None, "sm_max_mhz": mx, "samples": len(sm),
                "reasons": sorted(reasons), "source": "nvidia-smi"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_0801_1524_b200 as sft
    from paper_0801_1524_b200.dist import DistPlan

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    w = synth.make_workload(args.config)
    P = w.P
    prec = 1 if args.precision == "f32" else 0
    x = torch.from_numpy(w.x).to(dev)
    k = torch.from_numpy(w.k).to(dev)
    f = torch.from_numpy(w.f).to(dev)
    u = torch.empty(len(w.x), dtype=torch.complex128, device=dev)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def step():
        if world == 1:
            with sft.Plan(w.dim, w.N, w.p, x, k, stream=stream, precision=prec) as plan:
                plan.apply(f, u)
        else:
            with DistPlan(w.dim, w.N, w.p, x, k, stream=stream, exchange=args.exchange) as dp:
                dp.apply(f, u)

    def timed(fn, K, do_flush=True):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
        barrier()
        for i in range(K):
            if do_flush:
                flush.zero_()
            evs[i][0].record(stream)
            fn()
            evs[i][1].record(stream)
        torch.cuda.synchronize(dev)
        ms = [a.elapsed_time(b) for a, b in evs]
        tot = torch.tensor([sum(ms)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(tot, op=dist.ReduceOp.MAX)
        return float(tot.item()), ms

    for _ in range(args.warmup):
        step()
    launches0 = sft.launch_count()
    clk = Clocks(local)
    clk.start()
    total_ms, per_step = timed(step, args.steps)
    clocks = clk.stop()
    launches = sft.launch_count() - launches0

    # apply-only timing (plan reused) and per-kernel timing, same stream
    if world == 1:
        plan = sft.Plan(w.dim, w.N, w.p, x, k, stream=stream, precision=prec)
        for _ in range(max(2, args.warmup)):
            plan.apply(f, u)
        apply_total, _ = timed(lambda: plan.apply(f, u), args.steps)
        plan.set_timing(True)
        kt = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            plan.apply(f, u)
            torch.cuda.synchronize(dev)
            kt.append(plan.last_timing())
        # the translation chain as one interval (events around the first and last
        # translation launch only: the programmatic-dependent-launch overlap
        # between levels, which per-launch events cut, is kept) -- the roofline's
        # mean launch duration = chain / launches
        plan.set_timing(2)
        kc = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            plan.apply(f, u)
            torch.cuda.synchronize(dev)
            kc.append(plan.last_timing())
        plan.set_timing(False)
        st = plan.stats()
        work = plan.work()
        # multi-RHS apply (sft_apply_batch): args.nrhs
        # charge vectors through the plan, one launch per step for all of them;
        # skipped when the batch's level buffers would not fit comfortably
        batch = None
        R = args.nrhs
        need = R * st["level_buffer_bytes"]
        if R > 1 and need < 0.5 * torch.cuda.get_device_properties(dev).total_memory:
            F = torch.stack([torch.from_numpy(synth.random_charges(len(w.k), 1000 + r)) for r in range(R)]).to(dev)
            U = torch.empty(R, len(w.x), dtype=torch.complex128, device=dev)
            for _ in range(max(2, args.warmup)):
                plan.apply_batch(F, U)
            b_total, _ = timed(lambda: plan.apply_batch(F, U), args.steps)
            b_ms = b_total / args.steps
            batch = {"nrhs": R, "apply_ms": round(b_ms, 4), "apply_ms_per_rhs": round(b_ms / R, 4),
                     "mpoints_s": round(P * R / (b_ms / 1e3) / 1e6, 3),
                     "speedup_vs_single": round((apply_total / args.steps) * R / b_ms, 3),
                     "note": "f resident in HBM, L2 flushed before each batch; value = P * nrhs / batch apply time"}
            del F, U
        elif R > 1:
            batch = {"nrhs": R, "skipped": f"level buffers {need / 1e9:.1f} GB"}
        plan.close()
    else:
        dp = DistPlan(w.dim, w.N, w.p, x, k, stream=stream, exchange=args.exchange)
        for _ in range(max(2, args.warmup)):
            dp.apply(f, u)
        apply_total, _ = timed(lambda: dp.apply(f, u), args.steps)
        part = dp.partition().tolist()
        # this rank's translation time (both phases, CUDA events), max over ranks
        dp.plan.set_timing(True)
        tr = []
        for _ in range(max(3, min(args.steps, 10))):
            flush.zero_()
            dp.apply(f, u)
            torch.cuda.synchronize(dev)
            tr.append(dp.plan.last_timing()["trans_ms"])
        dp.plan.set_timing(False)
        trans_rank = torch.tensor([float(np.median(tr))], dtype=torch.float64, device=dev)
        dist.all_reduce(trans_rank, op=dist.ReduceOp.MAX)
        dist_trans_ms = float(trans_rank.item())
        dp.close()
        kt = None
        batch = None
        st = sft.Plan(w.dim, w.N, w.p, x, k, stream=stream)
        stats = st.stats()
        st.close()
        st = stats

    # end to end through the public API with pinned host buffers
    xh = torch.from_numpy(w.x).pin_memory()
    kh = torch.from_numpy(w.k).pin_memory()
    fh = torch.from_numpy(w.f).pin_memory()
    uh = torch.empty(len(w.x), dtype=torch.complex128).pin_memory()

    def step_e2e():
        if world == 1:
            with sft.Plan(w.dim, w.N, w.p, xh, kh, stream=stream, precision=prec) as plan:
                plan.apply(fh, uh)
        else:
            xd, kd, fd = xh.to(dev, non_blocking=True), kh.to(dev, non_blocking=True), fh.to(dev, non_blocking=True)
            with DistPlan(w.dim, w.N, w.p, xd, kd, stream=stream, exchange=args.exchange) as dp:
                ud = dp.apply(fd)
            uh.copy_(ud)

    for _ in range(2):
        step_e2e()
    e2e_total, _ = timed(step_e2e, args.steps)

    res = None
    if rank == 0:
        K = args.steps
        step_ms = total_ms / K
        value = P * K / (total_ms / 1e3) / 1e6
        hbm_peak, peak_src = measured_peaks()
        roof = None
        if kt:
            trans_lev_ms = float(np.median([t["trans_ms"] for t in kt]))
            trans_ms = float(np.median([t["trans_ms"] for t in kc]))
            leaf_ms = float(np.median([t["leaf_ms"] for t in kt]))
            final_ms = float(np.median([t["final_ms"] for t in kt]))
            app_ms = float(np.median([t["apply_ms"] for t in kt]))
            L = int(st["L"])
            nlaunch = len(st.get("launches", [])) or L
            # achieved = algorithmic (level-synchronous) bytes of all levels / the
            # launches' total device time (= per-launch bytes / mean launch duration)
            bytes_per_launch = st["trans_alg_bytes"] / nlaunch
            dur_per_launch = trans_ms / nlaunch / 1e3
            achieved = bytes_per_launch / dur_per_launch / 1e9
            traffic = None
            tf = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
            if os.path.exists(tf):
                traffic = json.load(open(tf)).get("dram_bytes_per_launch")
            n2 = sum(1 for _, f2 in st.get("launches", []) if f2)
            kname = "k_translate_ws (one launch per level" + (f", {n2} two-level launch)" if n2 else ")")
            f64p, f64src = fp64_peak()
            fl = work["fp64_flops"]
            fp64 = {"achieved": round(fl / (trans_ms / 1e3) / 1e12, 3), "peak": f64p, "unit": "TFLOP/s",
                    "frac": round(fl / (trans_ms / 1e3) / 1e12 / f64p, 4), "flops_per_apply": fl,
                    "supertiles": work["supertiles"], "peak_source": f64src,
                    "note": "FP64 flops the translation kernels execute (DMMA tiles whole incl. padding, plus "
                            "DADD/DMUL/DFMA; counted from the tile schedules, sft_plan_work) / translate ms"}
            roof = {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1), "fp64": fp64,
                    "peak": hbm_peak, "unit": "GB/s", "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                    "peak_source": peak_src,
                    "alg_bytes_per_launch": bytes_per_launch, "launches_per_apply": nlaunch,
                    "timing": "achieved = alg_bytes_per_launch / (translation chain ms / launches_per_apply); "
                              "chain = CUDA events before the first and after the last translation launch of an "
                              "apply (L2 flushed before each apply); translate_per_level_events = the sum of "
                              "per-launch event intervals (events between launches cut the PDL overlap)",
                    "achieved_per_level_events": round(bytes_per_launch / (trans_lev_ms / nlaunch / 1e3) / 1e9, 1),
                    "kernel_ms": {"leaf": round(leaf_ms, 4), "translate_total": round(trans_ms, 4),
                                  "translate_per_level_events": round(trans_lev_ms, 4),
                                  "final": round(final_ms, 4), "apply_events": round(app_ms, 4)},
                    "level_ms": [round(float(v), 4) for v in np.median([t["level_ms"] for t in kt], axis=0)]}
        if kt is None and world > 1:
            # sharded transform: all levels' algorithmic bytes over the slowest rank's
            # translation time, against the aggregate HBM peak of the N GPUs
            achieved = st["trans_alg_bytes"] / (dist_trans_ms / 1e3) / 1e9
            roof = {"bound": "hbm", "kernel": "k_translate_ws (all ranks, both phases)",
                    "achieved": round(achieved, 1), "peak": hbm_peak * world, "unit": "GB/s",
                    "frac": round(achieved / (hbm_peak * world), 4), "traffic": None, "peak_source": peak_src,
                    "note": f"aggregate over {world} GPUs: sum of level bytes / max-over-ranks translation ms",
                    "kernel_ms": {"translate_max_over_ranks": round(dist_trans_ms, 4)}}
        h2d = w.x.nbytes + w.k.nbytes + w.f.nbytes
        d2h = len(w.x) * 16
        res = {
            "metric": "butterfly SFT Mpoints/s (P=max(nx,nk) per plan+apply step)",
            "value": round(value, 3),
            "unit": "Mpoints/s",
            "n_gpus": world,
            "steps": K,
            "warmup": args.warmup,
            "ms_per_step": round(step_ms, 4),
            "apply_ms": round(apply_total / K, 4),
            "apply_mpoints_s": round(P * K / (apply_total / 1e3) / 1e6, 3),
            "plan_ms": round(step_ms - apply_total / K, 4),
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": args.precision,
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {CONFIG_DESC[args.config]}", "dim": w.dim, "N": w.N, "p": w.p,
                       "nx": len(w.x), "nk": len(w.k), "P": P, "pairs_total": int(np.sum(st["pairs"])),
                       "l2": "flushed before every timed step (256 MiB memset, outside the step events)",
                       "parallelism": (f"subtree-sharded x{world}, exchange {args.exchange}" if world > 1 else "single GPU")},
            "e2e": {"value": round(P * K / (e2e_total / 1e3) / 1e6, 3), "unit": "Mpoints/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": round(e2e_total / K, 4)},
            "gpu_launches": int(launches),
            "clocks": clocks,
            "roofline": roof,
        }
        if batch is not None:
            res["batch"] = batch
        if world > 1:
            res["partition"] = part[:3]
    if res is not None:
        # the GPU result of the last timed step (host copy, outside every timed region),
        # checked against the oracle in the cpu_baseline leg
        res["_u"] = u.cpu().numpy()
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return res, w


def cpu_baseline(w, nthreads=0, u_gpu=None):
    """The oracle (as it stands) on the host cores: the full oracle butterfly
    (the reported baseline), and the oracle direct sum on the seeded error
    sample, timed, with T_d -- the direct sum over all n_x targets -- estimated
    by scaling with n_x / sample size as the paper does (PAPER.md:383-389,
    "T_d ... estimated").  With the GPU's result u_gpu it also returns the
    accuracy of the benched run (BASELINE.json's metric includes the relative
    L2 error vs the direct sum): vs the oracle direct sum on the error sample
    (1024 seeded targets for C2/C4, BASELINE.json:9,11; all targets otherwise)
    and vs the oracle butterfly on every target."""
    import oracle
    nth = nthreads or oracle.max_threads()
    t0 = time.perf_counter()
    ub = oracle.butterfly(w.x, w.k, w.f, w.N, w.p, nthreads=nth)
    dt = time.perf_counter() - t0
    tg = w.sample if len(w.x) > 20000 else None
    t1 = time.perf_counter()
    ud = oracle.direct(w.x, w.k, w.f, w.N, targets=tg, nthreads=nth)
    dd = time.perf_counter() - t1
    t_d = dd * len(w.x) / len(ud)
    out = {"value": round(w.P / dt / 1e6, 6), "unit": "Mpoints/s", "cores": nth, "kind": "oracle",
           "cpu_model": cpu_model(),
           "sample": f"full {w.name} workload, one oracle butterfly (long double, OpenMP)",
           "seconds": round(dt, 3),
           "direct": {"targets": int(len(ud)), "seconds": round(dd, 3), "t_d_estimated_s": round(t_d, 2),
                      "note": "oracle direct sum (long double) on the error sample, T_d scaled by n_x / targets "
                              "(PAPER.md:386-389)"}}
    acc = None
    if u_gpu is not None:
        tol = {5: 5e-2, 7: 1e-3, 9: 1e-5}[w.p]
        ug = u_gpu if tg is None else u_gpu[tg]
        rms = lambda r: float(np.sqrt(np.mean(np.abs(r) ** 2)))  # noqa: E731
        acc = {"rel_l2_vs_direct": float(oracle.rel_l2(ug, ud)),
               "max_rel_vs_direct": float(np.max(np.abs(ug - ud)) / rms(ud)),
               "direct_targets": int(len(ud)), "direct_tol": tol,
               "rel_l2_vs_oracle_butterfly": float(oracle.rel_l2(u_gpu, ub)),
               "max_rel_vs_oracle_butterfly": float(np.max(np.abs(u_gpu - ub)) / rms(ub)), "parity_tol": 1e-10}
    return out, acc


def configs_block(steps=5, warmup=3):
    """Every BASELINE config (C0-C4) on this GPU: plan+apply step and apply
    time (CUDA events, L2 flushed), translation time and its HBM / FP64
    roofline fractions, and the relative L2 error vs the oracle direct sum on
    the seeded error sample (all targets for C0/C1; 1024 seeded targets for
    C2-C4 -- C3's all-target error is in tests/test_gpu_parity.py)."""
    import torch
    import oracle
    import paper_0801_1524_b200 as sft
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    hbm, _ = measured_peaks()
    f64p, _ = fp64_peak()
    out = {}
    for name in ("C0", "C1", "C2", "C3", "C4"):
        w = synth.make_workload(name)
        x = torch.from_numpy(w.x).to(dev); k = torch.from_numpy(w.k).to(dev); f = torch.from_numpy(w.f).to(dev)
        u = torch.empty(len(w.x), dtype=torch.complex128, device=dev)

        def step():
            with sft.Plan(w.dim, w.N, w.p, x, k, stream=stream) as pl:
                pl.apply(f, u)

        def timed(fn):
            ms = []
            for _ in range(steps):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream); fn(); b.record(stream)
                torch.cuda.synchronize(dev)
                ms.append(a.elapsed_time(b))
            return float(np.median(ms))
        for _ in range(warmup):
            step()
        step_ms = timed(step)
        pl = sft.Plan(w.dim, w.N, w.p, x, k, stream=stream)
        for _ in range(2):
            pl.apply(f, u)
        apply_ms = timed(lambda: pl.apply(f, u))
        pl.set_timing(2)  # the translation chain as one interval (as the main roofline)
        tr = []
        for _ in range(3):
            flush.zero_()
            pl.apply(f, u)
            torch.cuda.synchronize(dev)
            tr.append(pl.last_timing()["trans_ms"])
        trans_ms = float(np.median(tr))
        wk = pl.work()
        pl.close()
        ug = u.cpu().numpy()
        tg = synth.error_sample(len(w.x), w.seed) if len(w.x) > 20000 else None
        ud = oracle.direct(w.x, w.k, w.f, w.N, targets=tg)
        ugs = ug if tg is None else ug[tg]
        out[name] = {"step_ms": round(step_ms, 4), "mpoints_s": round(w.P / step_ms / 1e3, 3),
                     "apply_ms": round(apply_ms, 4), "translate_ms": round(trans_ms, 4),
                     "hbm_frac": round(wk["alg_bytes"] / (trans_ms / 1e3) / 1e9 / hbm, 4),
                     "fp64_frac": round(wk["fp64_flops"] / (trans_ms / 1e3) / 1e12 / f64p, 4),
                     "rel_l2_vs_direct": float(oracle.rel_l2(ugs, ud)), "direct_targets": int(len(ud))}
        del x, k, f, u
    return out


def _pairs(w, targets=None):
    L = w.N.bit_length() - 1

    def counts(pts):
        leaf = np.minimum(np.floor(pts).astype(np.int64), w.N - 1)
        mult = np.array([1 << (2 * L), 1 << L, 1][-w.dim:])
        return [len(np.unique((leaf >> (L - l)) @ mult)) for l in range(L + 1)]
    cx = counts(w.x if targets is None else w.x[targets])
    ck = counts(w.k)
    return sum(ck[t] * cx[L - t] for t in range(L + 1))


def run_reference(args):
    """--impl reference: the oracle on the host cores, rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle
    w = synth.make_workload(args.config)
    nth = oracle.max_threads()
    step = max(1, len(w.sample) // args.ref_targets)
    tg = w.sample[::step][: args.ref_targets]  # spread over the whole curve / surface
    frac = _pairs(w, tg) / _pairs(w)

    def step():
        oracle.butterfly(w.x, w.k, w.f, w.N, w.p, targets=tg, nthreads=nth)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    # full-workload equivalent: the oracle's cost is proportional to the pairs it visits
    value = w.P * frac / dt / 1e6
    desc = (f"oracle butterfly on {w.name} restricted to {len(tg)} seeded targets spread over the workload (all "
            f"sources): {frac:.4f} of the pairs; value = P * frac / step time.  The restricted run is cheaper per "
            f"pair than the full one (round 1 on C2: 0.0141 vs 0.0067 Mpoints/s for the full oracle in "
            f"cpu_baseline), so this overstates the oracle ~2x")
    return {
        "impl": "reference",
        "metric": "butterfly SFT Mpoints/s (P=max(nx,nk) per plan+apply step)",
        "value": round(value, 6),
        "unit": "Mpoints/s",
        "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64 (long double arithmetic)",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: {CONFIG_DESC[args.config]}", "dim": w.dim, "N": w.N, "p": w.p,
                   "nx": len(w.x), "nk": len(w.k), "P": w.P},
        "cpu_baseline": {"value": round(value, 6), "unit": "Mpoints/s", "cores": nth, "kind": "oracle",
                         "sample": desc},
        "e2e": {"value": round(value, 6), "unit": "Mpoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2", choices=sorted(CONFIG_DESC))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config block (C0-C4 on this GPU)")
    ap.add_argument("--ref-targets", type=int, default=256)
    ap.add_argument("--exchange", default="nccl", choices=["nccl", "fused", "torch"],
                    help="N > 1: level-m exchange and u all-gather by libsft's own NCCL calls (default), fused into "
                         "the exchange level's kernel (peer stores into IPC-mapped receive buffers over NVLink), or "
                         "torch.distributed collectives around the phase calls")
    ap.add_argument("--nrhs", type=int, default=4,
                    help="N = 1: also time sft_apply_batch with this many charge vectors (1 = skip)")
    ap.add_argument("--precision", default="f64", choices=["f64", "f32"],
                    help="arithmetic of the level charges (f32: the optional FP32 variant, single GPU)")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torchrun (the driver launches us that way itself)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world_env = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "ours" and world_env != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world_env}")
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        res = run_reference(args)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    res, w = run_ours(args)
    if res is not None:
        if res["n_gpus"] == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"], acc = cpu_baseline(w, u_gpu=res.get("_u"))
            if acc is not None:
                res["accuracy"] = acc
        if res["n_gpus"] == 1 and not args.no_cpu_baseline and not args.no_configs:
            res["configs"] = configs_block()
        res.pop("_u", None)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
