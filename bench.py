"""Benchmark of the Nystrom-Schur block-CG hot path (BASELINE.json metric:
"Schur block-CG: S_G X RHS-applies/s, time-to-tol, HBM GB/s vs peak").

One step = one pass of the whole hot path over one
batch of synthetic input:  B = K_G Omega (a0);  breakdown-free block CG on
S_G X = B to tol (a1-a11, M = I: the north_star-literal mode, every iteration is
exactly one S_G apply on n_G x s);  Y = A_G X (a12).
value = s * (block-CG iterations) / (step time)  [S_G RHS-applies per second],
whole job (one global problem sharded over the ranks).  Inputs resident in HBM
when the timed region starts; L2 flushed (256 MiB write) before every timed step.

Workload: BASELINE.json configs[4] (cfg5, 256^3 Laplacian, n = 16.8M, K = 1024,
s = 128) - the largest configuration and the one the north_star's scaling target
names; it fits one B200 (~130 GB).  The line also carries the paper-analog
M = A_G^-1 time-to-tol (reading C2), the Nystrom (Alg. 2) and outer-PCG (M_2 to
1e-8) times, the setup time, and a secondary object for cfg2 (configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Schur block-CG: S_G*X RHS-applies/s, time-to-tol, HBM GB/s vs peak"
UNIT = "RHS-applies/s"
FP64_PEAK_TFLOPS = 37.05  # DMMA m8n8k4 microbenchmark, tools/fp64_peak.cu -> profiles/r01_fp64_peak.txt


def _traffic(workload, kernel="k_symm"):
    """dram bytes per launch of the dominant kernel from one committed `ncu --set full` capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            t = json.load(f).get(workload)
        return (t["dram_bytes_per_launch"], t["source"]) if t and t.get("kernel") == kernel else (None, None)
    except Exception:
        return None, None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """SM clocks / throttle reasons sampled DURING the timed region: NVML polled every 5 ms from a
    thread (nvidia-smi -lms 100 as the fallback when pynvml is unavailable)."""

    def __init__(self, device=0):
        self.device = device
        self.proc = None
        self.lines = []
        self.nv = None
        self.samples = []      # (sm_mhz, reasons bitmask)
        self.max_mhz = None
        self.stop = threading.Event()

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:   # match the CUDA device by PCI bus id (CUDA_VISIBLE_DEVICES may renumber)
            import torch
            pr = torch.cuda.get_device_properties(self.device)
            bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.device)

    def _poll(self):
        nv, h = self.nv
        while not self.stop.is_set():
            try:
                self.samples.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                     nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            self.stop.wait(0.005)

    def __enter__(self):
        try:
            self.nv = self._nvml_handle()
            nv, h = self.nv
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nv = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap", "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], self.max_mhz, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        if self.nv is not None:
            bits = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
                    "sw_power_cap": 0x4}
            for mhz, r in self.samples:
                sm.append(float(mhz))
                for nm, b in bits.items():
                    if r & b:
                        reasons.add(nm)
            src = "nvml 5 ms"
        else:
            for ln in self.lines:
                p = [x.strip() for x in ln.split(",")]
                if len(p) < 7:
                    continue
                try:
                    sm.append(float(p[0]))
                    mx = float(p[1])
                except ValueError:
                    continue
                for nm, v in zip(names, p[3:7]):
                    if v.lower() == "active":
                        reasons.add(nm)
            src = "nvidia-smi 100 ms"
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm), "source": src}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _sample_blocks(K, nsample):
    """Evenly spread block ids of the bounded CPU sample (the extrapolation is linear in K)."""
    if nsample >= K:
        return list(range(K))
    return sorted(set(int(round(i * K / nsample)) for i in range(nsample)))


# ------------------------------------------------------------------------------------------
# the CPU oracle on a bounded sample (reference arm and cpu_baseline leg)
# ------------------------------------------------------------------------------------------
class OracleSample:
    """The oracle's S_G apply (oracle.SchurOracle: A_G X minus the per-block K_G terms with scipy
    SuperLU block solves), as it stands, on every core of this job's affinity mask (the block loop is
    spread over threads; SuperLU releases the GIL).  For K > nsample blocks the K_G sum is timed on an
    evenly spread sample of `nsample` blocks and extrapolated linearly:
        t_apply = t(A_G X) + (K / nsample) * t(K_G terms of the sample blocks)."""

    def __init__(self, pr, nsample):
        import oracle as O
        self.cores = _cores()
        self.pr = pr
        self.blocks = _sample_blocks(pr.K, nsample)
        t0 = time.perf_counter()
        self.d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K, blocks=None if len(self.blocks) == pr.K else self.blocks)
        self.S = O.SchurOracle(self.d, threads=self.cores)
        from oracle.schur import _map
        _map(self.S.lu_block, self.blocks, self.cores)      # factorisation: setup, not timed
        self.t_setup = time.perf_counter() - t0
        self.X = pr.omega()

    def apply_time(self):
        t0 = time.perf_counter()
        self.d.A_G @ self.X
        t1 = time.perf_counter()
        self.S.k_gamma(self.X, blocks=self.blocks)
        t2 = time.perf_counter()
        return (t1 - t0) + (t2 - t1) * self.pr.K / len(self.blocks)

    def describe(self):
        full = len(self.blocks) == self.pr.K
        return (f"one oracle S_G apply (s={self.pr.s}) on {self.pr.name} (n_G={self.d.n_gamma}, K={self.pr.K}): "
                f"A_G X plus the K_G terms of " + ("all blocks" if full else
                f"{len(self.blocks)} evenly spread blocks, extrapolated x{self.pr.K / len(self.blocks):.0f} "
                f"(linear in K)") + f"; scipy SuperLU block solves on {self.cores} threads ({_cpu_model()}); "
                f"block factorisation ({self.t_setup:.1f} s incl. extraction) untimed")


def run_reference(args, ws, rank):
    """bench.py --impl reference: the oracle as it stands on this box's host cores, same config /
    metric / unit; each step = one (bounded, extrapolated) oracle S_G apply.  Rank 0 only."""
    if rank != 0:
        return
    from nsp_inputs import problems as P
    pr = P.make(args.config)
    smp = OracleSample(pr, args.cpu_blocks)
    for _ in range(args.warmup):
        smp.apply_time()
    times = [smp.apply_time() for _ in range(args.steps)]
    tmean = sum(times) / len(times)
    value = pr.s / tmean
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tmean * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config, "s": pr.s, "n_gamma": smp.d.n_gamma,
                                            "K": pr.K, "parallelism": f"cpu-oracle {smp.cores} threads"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": smp.cores, "kind": "oracle",
                             "cpu_model": _cpu_model(), "sample": smp.describe()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(pr, seconds, nsample):
    """The oracle timed on a bounded sample of the same workload, all affinity cores."""
    smp = OracleSample(pr, nsample)
    smp.apply_time()
    t0 = time.perf_counter()
    ts = []
    while time.perf_counter() - t0 < seconds or not ts:
        ts.append(smp.apply_time())
    t = sum(ts) / len(ts)
    return {"value": pr.s / t, "unit": UNIT, "cores": smp.cores, "kind": "oracle", "cpu_model": _cpu_model(),
            "sample": f"{len(ts)} x " + smp.describe()}


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
def _timed(stream, fn, flush, reps):
    import torch
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    out = []
    for _ in range(reps):
        flush.zero_()
        ev0.record(stream)
        r = fn()
        ev1.record(stream)
        torch.cuda.synchronize()
        out.append((ev0.elapsed_time(ev1), r))
    return out


def measure(pr, args, ws, rank, local, stream, nccl_id, headline):
    """Time one configuration; returns the dict of measurements (headline: the full set)."""
    import torch
    from paper_2101_12164_b200 import nsp
    dev = torch.device("cuda", local)
    single = ws == 1
    t0 = time.perf_counter()
    ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, device=local,
                      stream=stream.cuda_stream, nranks=ws, rank=rank, nccl_id=nccl_id,
                      factor_gamma=single)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    st = ctx.stats()
    s, nG = pr.s, ctx.n_gamma_local
    pos = np.searchsorted(pr.gamma, ctx.gamma_index())      # local Gamma rows of this rank
    Om_h = torch.from_numpy(np.ascontiguousarray(pr.omega()[pos])).pin_memory()
    Om = Om_h.to(dev)
    Bm = torch.empty(nG, s, dtype=torch.float64, device=dev)
    X = torch.empty_like(Bm)
    Y = torch.empty_like(Bm)
    Y_h = torch.empty(nG, s, dtype=torch.float64).pin_memory()
    wsbuf = torch.empty(ctx.workspace_bytes(s), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    maxit = args.maxit
    out = {"workload": pr.name, "n": pr.n, "n_gamma": ctx.n_gamma, "n_gamma_local": nG, "K": pr.K, "s": s,
           "tol_bcg": pr.tol_bcg, "setup_ms": t_setup * 1e3,
           "setup_split_ms": dict(zip(["host_analysis", "h2d", "gpu_factor", "ag_operator", "sj_inverse_tiles",
                                       "sj_inverse_int8_slices"], ctx.setup_report["t_ms"][:6])),
           "shared_rows": ctx.n_shared}

    def step():
        ctx.kgamma_apply(Om, Bm, wsbuf)
        rep = ctx.block_cg(Bm, X, pr.tol_bcg, maxit, wsbuf)
        ctx.gamma_apply(X, Y)
        return rep

    ctx.set_bcg_precond(0)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    launches0 = nsp.kernel_launches()
    with ClockSampler(local) as clk:
        if ws > 1:
            torch.distributed.barrier()
        res = _timed(stream, step, flush, args.steps)
        if ws > 1:
            torch.distributed.barrier()
    out["clocks"] = clk.summary()
    out["gpu_launches"] = (nsp.kernel_launches() - launches0) / args.steps
    fr_, tot_ = torch.cuda.mem_get_info(dev)
    out["device_memory_gb"] = {"in_use": (tot_ - fr_) / 1e9, "total": tot_ / 1e9}
    times = [t for t, _ in res]
    iters = [r["iters"] for _, r in res]
    tmean = sum(times) / len(times)
    if ws > 1:
        tt = torch.tensor([tmean], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        tmean = float(tt.item())
    it_mean = sum(iters) / len(iters)
    out.update(time_to_tol_ms=tmean, bcg_iters=it_mean, bcg_precond="none (M = I)",
               rhs_applies_per_s=s * it_mean / (tmean * 1e-3), iteration_ms=tmean / max(it_mean, 1))
    # live duration of the dominant kernel (a2+a3, k_symm): the same steps with a CUDA event pair around
    # every a2+a3 launch on the context stream (per-iteration graphs carry the pair)
    ctx.profile(True)
    ctx.profile_read()
    pc0 = nsp.path_counters()
    for _ in range(min(args.steps, 3)):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    sweep_ms, sweeps = ctx.profile_read()
    ctx.profile(False)
    int8 = nsp.path_counters()["ozaki"] > pc0["ozaki"]
    # tile bookkeeping: stored lower S_j^-1 tiles T_l = sum ntb(ntb+1)/2, W/V/U tiles T_w = sum ntb,
    # (output tile, K tile) pairs sum ntb^2 = 2 T_l - T_w
    t_l, t_w = st["l22_entries"] // 4096, st["wvu_rows"] // 64
    nct = (s + 127) // 128
    oz = ctx.ozaki_stats()
    # share of the 28 slice products per (unit, K tile) that k_oz_symm executes: the products with an all-zero
    # leading S_j^-1 slice are skipped (exact zeros), so they are not counted as work either
    keep = oz["slice_products_executed"] / oz["slice_products_full"] if oz["slice_products_full"] else 1.0
    out["k_symm"] = {"avg_launch_ms": sweep_ms / max(sweeps, 1), "launches": sweeps,
                     "flops_per_launch": 2.0 * st["sum_b2"] * s, "int8": int8,
                     # INT8 path, algorithmic: the exact int8 slice products per fp64 multiply-add of
                     # U_j = S_j^-1 W_j (2 s sum b_j^2 of them) - 28, times the executed share `keep` (the
                     # leading-zero-slice skip); the tiles' zero padding, +2.3 % at cfg5, is not counted
                     "int8_ops_per_launch": 28 * keep * 2.0 * st["sum_b2"] * s,
                     "int8_ops_28_products_per_launch": 28 * 2.0 * st["sum_b2"] * s,
                     "int8_products_kept": keep,
                     "int8_ops_executed_per_launch": 2.0 * 128 * 64 * 64 * oz["slice_products_executed"] * nct,
                     # unique bytes: the stored tiles' slices (skip applied), the W^T slices, U out (fp64)
                     "int8_alg_bytes_per_launch": (oz["m_slice_bytes"] or 7 * 4096 * t_l) + 7 * 8192 * nct * t_w
                     + 8 * s * st["wvu_rows"],
                     "alg_bytes_per_launch": 8 * (st["sum_b2"] + st["sum_b"]) / 2 + 2 * 8 * s * st["sum_b"]}
    # apply-only timing (a1-a5), L2 flushed
    P_ = torch.randn(nG, s, dtype=torch.float64, device=dev)
    Q_ = torch.empty_like(P_)
    at = [t for t, _ in _timed(stream, lambda: ctx.schur_apply(P_, Q_, wsbuf), flush, args.apply_reps + 3)[3:]]
    t_apply = statistics.median(at)
    tg = [t for t, _ in _timed(stream, lambda: ctx.gamma_apply(P_, Q_), flush, args.apply_reps + 3)[3:]]
    t_gamma = statistics.median(tg)
    out["apply"] = {"ms": t_apply, "rhs_applies_per_s": s / (t_apply * 1e-3),
                    "a2a3_tflops": 2.0 * st["sum_b2"] * s / (t_apply * 1e-3) / 1e12, "gamma_apply_ms": t_gamma}
    # one block-CG iteration: the step minus its a0 (K_G Omega, one apply) and a12 (A_G X), per iteration
    it_ms = (out["time_to_tol_ms"] - t_apply - t_gamma) / max(out["bcg_iters"], 1)
    out["iteration_ms"] = it_ms
    out["iteration_split_ms"] = {"iteration": it_ms, "apply": t_apply, "grams_panels_sxs": it_ms - t_apply,
                                 "step_outside_loop": t_apply + t_gamma}
    # e2e: Omega from pinned host memory, Y back to pinned host memory, inside the timed region
    def step_e2e():
        Om.copy_(Om_h, non_blocking=True)
        r = step()
        Y_h.copy_(Y, non_blocking=True)
        return r
    et = _timed(stream, step_e2e, flush, max(1, args.steps))
    e2e_t = sum(t for t, _ in et) / len(et)
    if ws > 1:
        tt = torch.tensor([e2e_t], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        e2e_t = float(tt.item())
    e2e_it = sum(r["iters"] for _, r in et) / len(et)
    e2e_serial = s * e2e_it / (e2e_t * 1e-3)

    # e2e as a serving loop runs it: the same K steps back to back, double-buffered - step k + 1's Omega upload
    # (copy stream) overlaps step k's block CG, step k's Y download (second copy stream) overlaps step k + 1;
    # timed from the first upload's start to the last download's end (every step's copies inside the region)
    def e2e_pipelined(nsteps):
        Omb, Yb = [Om, torch.empty_like(Om)], [Y, torch.empty_like(Y)]
        Yhb = [Y_h, torch.empty_like(Y_h).pin_memory()]
        s_in, s_out = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
        e_in = [torch.cuda.Event(), torch.cuda.Event()]
        e_used = [torch.cuda.Event(), torch.cuda.Event()]
        e_y = [torch.cuda.Event(), torch.cuda.Event()]
        e_out = [torch.cuda.Event(), torch.cuda.Event()]
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flush.zero_()
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        t0.record(s_in)
        with torch.cuda.stream(s_in):
            Omb[0].copy_(Om_h, non_blocking=True)
        e_in[0].record(s_in)
        its = []
        for k in range(nsteps):
            b = k % 2
            stream.wait_event(e_in[b])
            if k >= 2:
                stream.wait_event(e_out[b])          # Y[b] downloaded before step k overwrites it
            ctx.kgamma_apply(Omb[b], Bm, wsbuf)
            e_used[b].record(stream)
            if k + 1 < nsteps:
                nb = 1 - b
                if k >= 1:
                    s_in.wait_event(e_used[nb])      # Omega[nb] consumed by step k - 1
                with torch.cuda.stream(s_in):
                    Omb[nb].copy_(Om_h, non_blocking=True)
                e_in[nb].record(s_in)
            r = ctx.block_cg(Bm, X, pr.tol_bcg, maxit, wsbuf)
            ctx.gamma_apply(X, Yb[b])
            e_y[b].record(stream)
            s_out.wait_event(e_y[b])
            with torch.cuda.stream(s_out):
                Yhb[b].copy_(Yb[b], non_blocking=True)
            e_out[b].record(s_out)
            its.append(r["iters"])
        t1.record(s_out)
        torch.cuda.synchronize()
        return t0.elapsed_time(t1), sum(its)
    e2e_pipelined(2)                                  # warm-up (second Y / Omega buffers, streams)
    tp, itp = e2e_pipelined(max(2, args.steps))
    if ws > 1:
        tt = torch.tensor([tp], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        tp = float(tt.item())
    out["e2e"] = {"value": s * itp / (tp * 1e-3), "unit": UNIT, "h2d_bytes_per_step": nG * s * 8,
                  "d2h_bytes_per_step": nG * s * 8,
                  "mode": "K steps back to back through the public API, double-buffered: step k+1's Omega upload "
                          "and step k's Y download (pinned host memory, two copy streams) overlap the compute; "
                          "timed from the first upload's start to the last download's end",
                  "serial_value": e2e_serial,
                  "serial_mode": "each step alone: upload, step, download, synchronize (L2 flushed between steps)"}
    if single and not args.no_analog:
        # the paper-analog block-CG preconditioner M = A_G^-1 (reading C2), same context
        ctx.set_bcg_precond(1)
        for _ in range(max(1, args.warmup - 1)):
            step()
        ra = _timed(stream, step, flush, args.steps)
        ta = sum(t for t, _ in ra) / len(ra)
        ia = sum(r["iters"] for _, r in ra) / len(ra)
        ctx.set_bcg_precond(0)
        out["paper_analog"] = {"bcg_precond": "A_G^-1 (paper-analog, reading C2; " +
                               ("Chebyshev A_G^-1" if st["ag_bw"] < 0 else "partitioned band factor") + ")",
                               "time_to_tol_ms": ta, "bcg_iters": ia, "rhs_applies_per_s": s * ia / (ta * 1e-3)}
    if single and not args.no_nystrom:
        # Nystrom (Alg. 2: B = K_G Omega, block CG to tol, Y = A_G X, CholQR2, EVDs, Z = A_G^-1 U) and the
        # outer PCG on the full system with M_2 to tol_pcg (eq:Sx=b)
        del wsbuf
        torch.cuda.empty_cache()
        ctx.nystrom(pr.rank, pr.oversample, Om, pr.tol_bcg, maxit)   # warm-up: workspaces, graph capture
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rn = ctx.nystrom(pr.rank, pr.oversample, Om, pr.tol_bcg, maxit)
        torch.cuda.synchronize()
        out["nystrom_ms"] = (time.perf_counter() - t0) * 1e3
        out["nystrom_inner_iters"] = rn["iters"]
        out["nystrom_rank"] = rn["rank"]
        b = torch.from_numpy(pr.rhs()).to(dev)
        xs = torch.zeros_like(b)
        tol_pcg = pr.tol_pcg or 1e-8
        ctx.pcg(b, xs, tol_pcg, 20000, precond=2)          # warm-up (graph capture)
        torch.cuda.synchronize()
        pt = []
        for _ in range(2):
            xs.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rp = ctx.pcg(b, xs, tol_pcg, 20000, precond=2)
            torch.cuda.synchronize()
            pt.append((time.perf_counter() - t0) * 1e3)
        out["pcg_ms"] = min(pt)
        out["pcg_iters"] = rp["iters"]
        out["pcg_tol"] = tol_pcg
        out["pcg_precond"] = "M_2 (Nystrom-Schur, Alg. 2)"
    ctx.close()
    return out


def run_ours(args, ws, rank, local):
    import torch
    from nsp_inputs import problems as P
    from paper_2101_12164_b200 import build as B
    from paper_2101_12164_b200 import nsp
    B.build()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)
    nccl_id = None
    if ws > 1:   # the library's own NCCL communicator; its unique id travels through the process group
        obj = [nsp.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    pr = P.make(args.config)
    m = measure(pr, args, ws, rank, local, stream, nccl_id, headline=True)
    peaks = _peaks()
    ks = m["k_symm"]
    achieved = ks["flops_per_launch"] / (ks["avg_launch_ms"] * 1e-3) / 1e12
    if ks["int8"]:
        traffic, traffic_src = _traffic(args.config + "_int8", "k_oz_symm")
        i8_peak = 2.0 * peaks.get("bf16_tflops", 2250.0)
        i8_ach = ks["int8_ops_per_launch"] / (ks["avg_launch_ms"] * 1e-3) / 1e12
        roof = {"kernel": "k_oz_symm (a2+a3: U_j = S_j^-1 W_j on the INT8 tensor cores, tcgen05 kind::i8 with TMEM "
                          "accumulators; Ozaki splitting into 7 int8 slices, 28 exact int32 slice products, fp64 "
                          "result; reading R10)",
                "bound": "tensor", "achieved": i8_ach, "peak": i8_peak, "unit": "TOP/s", "frac": i8_ach / i8_peak,
                "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst, cuBLAS) x 2, the nominal INT8:BF16 dense "
                               "ratio of the B200 tensor core" + ("" if "bf16_tflops" in peaks else
                                                                  " (fallback: nominal 2.25 PF bf16)"),
                "algorithmic_int8_ops_per_launch": ks["int8_ops_per_launch"],
                "int8_products_kept": ks["int8_products_kept"],
                "int8_ops_28_products_per_launch": ks["int8_ops_28_products_per_launch"],
                "executed_int8_ops_per_launch": ks["int8_ops_executed_per_launch"],
                "algorithmic_bytes_per_launch": ks["int8_alg_bytes_per_launch"],
                "fp64_equivalent_tflops": achieved,
                "fp64_equivalent_vs_dmma_peak": achieved / FP64_PEAK_TFLOPS,
                "hbm_gbs_at_alg_bytes": ks["int8_alg_bytes_per_launch"] / (ks["avg_launch_ms"] * 1e-3) / 1e9}
    else:
        traffic, traffic_src = _traffic(args.config)
        roof = {"kernel": "k_symm (a2+a3: U_j = S_j^-1 W_j, all blocks one launch)", "bound": "tensor",
                "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "fp64 DMMA microbenchmark tools/fp64_peak.cu (profiles/r01_fp64_peak.txt); "
                               "MEASURED_PEAKS.json has no fp64 figure",
                "algorithmic_flops_per_launch": ks["flops_per_launch"],
                "algorithmic_bytes_per_launch": ks["alg_bytes_per_launch"],
                "hbm_gbs_at_alg_bytes": ks["alg_bytes_per_launch"] / (ks["avg_launch_ms"] * 1e-3) / 1e9}
    roof.update({"avg_launch_ms": ks["avg_launch_ms"], "launches": ks["launches"],
                 "timing": "CUDA events around each launch of the kernel on the context stream, in a pass of the "
                           "same steps right after the timed region (the timed region runs the event-free "
                           "device-driven loop graph)",
                 "hbm_peak_gbs": peaks.get("hbm_gbs"), "iteration_split_ms": m["iteration_split_ms"]})
    traffic, traffic_src = roof["traffic"], roof["traffic_source"]
    line = {
        "metric": METRIC, "value": m["rhs_applies_per_s"] * 1.0, "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": m["time_to_tol_ms"],
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "dtype_note": "fp64 results; a2+a3 as exact int32 sums of int8 slice products on the tensor cores (reading R10)",
        "data": "synthetic",
        "config": {"workload": args.config, "n": pr.n, "n_gamma": m["n_gamma"], "K": pr.K, "s": pr.s,
                   "tol_bcg": pr.tol_bcg, "bcg_precond": "none (M = I, north_star-literal)",
                   "parallelism": f"subdomains over {ws} ranks (contiguous ND subtrees, shared-separator NCCL "
                                  f"allreduce)" if ws > 1 else "1gpu",
                   "shared_rows": m["shared_rows"], "l2": "flushed (256 MiB write) before every timed step"},
        "time_to_tol_ms": m["time_to_tol_ms"], "bcg_iters": m["bcg_iters"],
        "paper_analog": m.get("paper_analog"),
        "nystrom_ms": m.get("nystrom_ms"), "nystrom_inner_iters": m.get("nystrom_inner_iters"),
        "pcg_ms": m.get("pcg_ms"), "pcg_iters": m.get("pcg_iters"), "pcg_tol": m.get("pcg_tol"),
        "setup_ms": m["setup_ms"], "setup_split_ms": m["setup_split_ms"],
        "apply": m["apply"], "iteration_split_ms": m["iteration_split_ms"],
        "roofline": roof,
        "e2e": m["e2e"], "gpu_launches": m["gpu_launches"], "clocks": m["clocks"],
        "device_memory_gb": m.get("device_memory_gb"),
    }
    if ws == 1 and not args.no_secondary and args.secondary and args.secondary != args.config:
        torch.cuda.empty_cache()
        pr2 = P.make(args.secondary)
        m2 = measure(pr2, args, ws, rank, local, stream, nccl_id, headline=False)
        line["secondary"] = {k: m2.get(k) for k in ("workload", "n", "n_gamma", "K", "s", "time_to_tol_ms",
                                                     "bcg_iters", "rhs_applies_per_s", "iteration_ms", "apply",
                                                     "paper_analog", "nystrom_ms", "nystrom_inner_iters",
                                                     "pcg_ms", "pcg_iters", "setup_ms", "e2e", "k_symm")}
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(pr, args.cpu_seconds, args.cpu_blocks)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()


def _relaunch(args):
    """bench.py --gpus N without torchrun: launch N ranks (one per GPU) through torch.distributed.run."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--secondary", default="cfg2", help="second workload reported in the same line (N = 1)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--maxit", type=int, default=1000)
    ap.add_argument("--apply-reps", type=int, default=10)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--cpu-blocks", type=int, default=16, help="blocks in the oracle's bounded timing sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-analog", action="store_true", help="skip the M = A_G^{-1} block-CG timing")
    ap.add_argument("--no-nystrom", action="store_true", help="skip the Nystrom + outer PCG timing")
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        _relaunch(args)
    ws, rank, local = _dist()
    if ws != args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={ws}"}), flush=True)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
