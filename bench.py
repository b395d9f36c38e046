"""Benchmark of the Nystrom-Schur block-CG hot path (BASELINE.json metric:
"Schur block-CG: S_G X RHS-applies/s, time-to-tol, HBM GB/s vs peak").

One step = one pass of the whole hot path over one
batch of synthetic input:  B = K_G Omega (a0);  breakdown-free block CG on
S_G X = B to tol (a1-a11);  Y = A_G X (a12).
value = s * (block-CG iterations) / (step time)  [S_G RHS-applies per second],
whole job (summed over ranks).  Inputs resident in HBM when the timed region
starts; L2 flushed (256 MiB write) before every timed step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg2] [--impl ours|reference]
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


# ------------------------------------------------------------------------------------------
# reference arm: the CPU oracle, as it stands, on this box's host cores
# ------------------------------------------------------------------------------------------
def run_reference(args, ws, rank):
    if rank != 0:
        return
    from threadpoolctl import threadpool_limits
    import oracle as O
    from nsp_inputs import problems as P
    pr = P.make(args.config)
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    s = pr.s
    X = pr.omega()
    with threadpool_limits(limits=1):
        t0 = time.perf_counter()
        for j in range(d.K):
            S.lu_block(j)                      # factorisation (not timed in the metric)
        t_fact = time.perf_counter() - t0
        for _ in range(args.warmup):
            S.apply(X)
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            S.apply(X)
            times.append(time.perf_counter() - t0)
    tmean = sum(times) / len(times)
    value = s / tmean
    sample = (f"one oracle S_G apply (scipy SuperLU per block, 1 thread) on {args.config} "
              f"(n_G={d.n_gamma}, s={s}) per step; block factorisation {t_fact:.1f}s untimed")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tmean * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": args.config, "s": s, "n_gamma": d.n_gamma,
                                            "parallelism": "cpu-oracle"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline(pr, seconds=20.0):
    """The oracle timed on a bounded sample: S_G applies on the same workload (1 thread)."""
    from threadpoolctl import threadpool_limits
    import oracle as O
    d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
    S = O.SchurOracle(d)
    X = pr.omega()
    with threadpool_limits(limits=1):
        for j in range(d.K):
            S.lu_block(j)
        S.apply(X)
        t0 = time.perf_counter()
        reps = 0
        while time.perf_counter() - t0 < seconds or reps == 0:
            S.apply(X)
            reps += 1
        t = (time.perf_counter() - t0) / reps
    return {"value": pr.s / t, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{reps} oracle S_G applies (s={pr.s}) on {pr.name}, scipy SuperLU block solves, "
                      f"1 thread; block factorisation untimed"}


# ------------------------------------------------------------------------------------------
# our arm
# ------------------------------------------------------------------------------------------
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
    pr = P.make(args.config)
    nccl_id = None
    if ws > 1:   # the library's own NCCL communicator; its unique id travels through the process group
        obj = [nsp.nccl_unique_id() if rank == 0 else None]
        torch.distributed.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    t0 = time.perf_counter()
    ctx = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, device=local,
                      stream=stream.cuda_stream, nranks=ws, rank=rank, nccl_id=nccl_id)
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

    def step():
        ctx.kgamma_apply(Om, Bm, wsbuf)
        rep = ctx.block_cg(Bm, X, pr.tol_bcg, maxit, wsbuf)
        ctx.gamma_apply(X, Y)
        return rep

    for _ in range(args.warmup):
        rep = step()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    launches0 = nsp.kernel_launches()
    times, iters = [], []
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # the timed region runs the production path (the device-driven loop graph, no per-kernel events)
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.zero_()
            ev0.record(stream)
            rep = step()
            ev1.record(stream)
            torch.cuda.synchronize()
            times.append(ev0.elapsed_time(ev1))
            iters.append(rep["iters"])
    launches = (nsp.kernel_launches() - launches0) / args.steps
    # live duration of the dominant kernel: the same K steps again with a CUDA event pair around every
    # a2+a3 launch on the context stream (the loop then runs as one graph per iteration, which carries
    # the event pair; the events bracket only that kernel)
    ctx.profile(True)
    ctx.profile_read()
    for _ in range(args.steps):
        flush.zero_()
        step()
    torch.cuda.synchronize()
    sweep_ms, sweeps = ctx.profile_read()
    ctx.profile(False)
    # apply-only timing (K1/K2 pipeline), same stream, L2 flushed
    P_ = torch.randn(nG, s, dtype=torch.float64, device=dev)
    Q_ = torch.empty_like(P_)
    at = []
    for i in range(args.apply_reps + 3):
        flush.zero_()
        ev0.record(stream)
        ctx.schur_apply(P_, Q_, wsbuf)
        ev1.record(stream)
        torch.cuda.synchronize()
        if i >= 3:
            at.append(ev0.elapsed_time(ev1))
    t_apply = statistics.median(at)
    # the same apply with the two batched L22 triangular sweeps (north_star (b) literal kernel)
    ctx_sw = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, device=local,
                         stream=stream.cuda_stream, nranks=ws, rank=rank, nccl_id=nccl_id, apply_kernel=1) \
        if ws == 1 else None
    t_apply_sweeps = None
    if ctx_sw is not None:
        ws_sw = torch.empty(ctx_sw.workspace_bytes(s), dtype=torch.uint8, device=dev)
        at2 = []
        for i in range(args.apply_reps + 3):
            flush.zero_()
            ev0.record(stream)
            ctx_sw.schur_apply(P_, Q_, ws_sw)
            ev1.record(stream)
            torch.cuda.synchronize()
            if i >= 3:
                at2.append(ev0.elapsed_time(ev1))
        t_apply_sweeps = statistics.median(at2)
        ctx_sw.close()
        del ws_sw
    # the paper-analog block-CG preconditioner M = A_G^{-1} (reading C2): same step, its own context
    analog = None
    if ws == 1 and not args.no_analog:
        ctx_a = nsp.Context(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, device=local,
                            stream=stream.cuda_stream, bcg_precond=1)
        ws_a = torch.empty(ctx_a.workspace_bytes(s), dtype=torch.uint8, device=dev)
        Ba, Xa, Ya = torch.empty_like(Bm), torch.empty_like(Bm), torch.empty_like(Bm)

        def step_a():
            ctx_a.kgamma_apply(Om, Ba, ws_a)
            r = ctx_a.block_cg(Ba, Xa, pr.tol_bcg, maxit, ws_a)
            ctx_a.gamma_apply(Xa, Ya)
            return r
        for _ in range(args.warmup):
            step_a()
        ta, ia = [], []
        for _ in range(args.steps):
            flush.zero_()
            ev0.record(stream)
            r = step_a()
            ev1.record(stream)
            torch.cuda.synchronize()
            ta.append(ev0.elapsed_time(ev1))
            ia.append(r["iters"])
        analog = {"bcg_precond": "A_G^-1 (paper-analog, reading C2)", "time_to_tol_ms": sum(ta) / len(ta),
                  "bcg_iters": sum(ia) / len(ia),
                  "rhs_applies_per_s": s * (sum(ia) / len(ia)) / (sum(ta) / len(ta) * 1e-3)}
        ctx_a.close()
        del ws_a
    # e2e: Omega from pinned host memory, Y back to pinned host memory, inside the timed region
    et = []
    for _ in range(max(1, args.steps)):
        flush.zero_()
        ev0.record(stream)
        Om.copy_(Om_h, non_blocking=True)
        rep_e = step()
        Y_h.copy_(Y, non_blocking=True)
        ev1.record(stream)
        torch.cuda.synchronize()
        et.append((ev0.elapsed_time(ev1), rep_e["iters"]))
    tmax = sum(times) / len(times)
    if ws > 1:
        tt = torch.tensor([tmax], device=dev)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        tmax = float(tt.item())
    it_mean = sum(iters) / len(iters)
    value = s * it_mean / (tmax * 1e-3)      # one global problem sharded over ws ranks (strong scaling)
    e2e_t = sum(t for t, _ in et) / len(et)
    e2e_it = sum(i for _, i in et) / len(et)
    e2e_val = s * e2e_it / (e2e_t * 1e-3)
    # roofline of the dominant kernel: the batched factor sweeps (a2+a3), fp64 DMMA-bound
    sweep_avg_ms = sweep_ms / max(sweeps, 1)
    flops_per_launch = 2.0 * st["sum_b2"] * s      # forward + backward: 2 * b_j^2 * s per block
    achieved = flops_per_launch / (sweep_avg_ms * 1e-3) / 1e12
    # algorithmic bytes: the unpadded lower triangle of every S_j^{-1} streamed once (k_symm: each
    # stored tile serves two output rows) + W in + U out (s-wide boundary-layer rows)
    hbm_alg = 8 * (st["sum_b2"] + st["sum_b"]) / 2 + 2 * 8 * s * st["sum_b"]
    peaks = _peaks()
    traffic, traffic_src = _traffic(args.config)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": tmax, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": args.config, "n": pr.n, "n_gamma": nG, "K": pr.K, "s": s,
                   "tol_bcg": pr.tol_bcg, "bcg_precond": "none",
                   "parallelism": f"subdomains{ws} (blocks per rank, shared-separator NCCL allreduce)" if ws > 1
                   else "1gpu", "n_gamma_global": ctx.n_gamma, "shared_rows": ctx.n_shared,
                   "l2": "flushed (256 MiB write) before every timed step"},
        "time_to_tol_ms": tmax, "bcg_iters": it_mean, "paper_analog": analog,
        "apply": {"ms": t_apply, "rhs_applies_per_s": s / (t_apply * 1e-3), "a2a3": "k_symm (explicit S_j^-1 tiles)",
                  "sweeps_ms": t_apply_sweeps,
                  "sweeps_rhs_applies_per_s": s / (t_apply_sweeps * 1e-3) if t_apply_sweeps else None},
        "roofline": {"kernel": "k_symm (a2+a3: U_j = S_j^-1 W_j, all blocks one launch)", "bound": "tensor",
                     "achieved": achieved, "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                     "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
                     "algorithmic_bytes_per_launch": hbm_alg,
                     "peak_source": "fp64 DMMA microbenchmark tools/fp64_peak.cu (profiles/r01_fp64_peak.txt)",
                     "algorithmic_flops_per_launch": flops_per_launch, "avg_launch_ms": sweep_avg_ms,
                     "timing": "CUDA events around each a2+a3 launch on the context stream, in a pass of the "
                               "same K steps right after the timed region (the timed region itself runs "
                               "the event-free device-driven loop graph)",
                     "launches": sweeps,
                     "hbm_gbs_at_alg_bytes": hbm_alg / (sweep_avg_ms * 1e-3) / 1e9,
                     "hbm_peak_gbs": peaks.get("hbm_gbs")},
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": nG * s * 8, "d2h_bytes_per_step": nG * s * 8},
        "gpu_launches": launches,
        "setup_s": t_setup, "setup_ms": ctx.setup_report["t_ms"][:3],
        "clocks": clk.summary(),
    }
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(pr, args.cpu_seconds)
    if rank == 0:
        print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        torch.distributed.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--maxit", type=int, default=1000)
    ap.add_argument("--apply-reps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=20.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-analog", action="store_true", help="skip the M = A_G^-1 block-CG timing")
    args = ap.parse_args()
    ws, rank, local = _dist()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    run_ours(args, ws, rank, local)


if __name__ == "__main__":
    main()
