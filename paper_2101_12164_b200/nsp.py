"""Thin ctypes binding of include/nsp.h (same names, argument marshalling only).

Device blocks are torch CUDA float64 tensors (PyTorch supplies device memory and
streams - plumbing, not compute); every step of the path runs in libnsp.so.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NSP_LIB") or os.path.join(_HERE, "libnsp.so")   # NSP_LIB: tuning variants only

NSP_STATUS = {0: "NSP_OK", 1: "NSP_NOT_CONVERGED", -1: "NSP_ERR_ARG", -2: "NSP_ERR_NOT_SPD",
              -3: "NSP_ERR_INDEFINITE", -4: "NSP_ERR_STAGNATION", -5: "NSP_ERR_RANK_COLLAPSE",
              -6: "NSP_ERR_NUMERICAL", -7: "NSP_ERR_STATE", -8: "NSP_ERR_CUDA", -9: "NSP_ERR_NCCL",
              -10: "NSP_ERR_OOM"}

EXPORTED = ["nsp_default_opts", "nsp_setup", "nsp_dims", "nsp_gamma_index", "nsp_workspace_bytes",
            "nsp_stats", "nsp_ozaki_stats", "nsp_schur_apply", "nsp_kgamma_apply", "nsp_block_cg", "nsp_nystrom",
            "nsp_nystrom_sigma", "nsp_precond_apply", "nsp_pcg", "nsp_last_error", "nsp_destroy",
            "nsp_gamma_apply", "nsp_kernel_launches", "nsp_profile", "nsp_profile_read", "nsp_shard_plan",
            "nsp_shard_info", "nsp_nccl_unique_id", "nsp_nccl_selftest", "nsp_local_group_create", "nsp_local_group_destroy",
            "nsp_set_bcg_precond", "nsp_path_counters", "nsp_dev_panel", "nsp_dev_gram", "nsp_dev_panel_gram",
            "nsp_dev_philox_gaussian", "nsp_dev_set_fused_pg"]

# dispatch-path counter ids (include/nsp.h NSP_PATH_*)
PATHS = ["panel_rows", "panel_tiles", "gram_sym", "gram_de", "gram_full", "symm", "sweeps", "symv",
         "panel_gram", "chol_solve", "ozaki"]


class nsp_csr(C.Structure):
    _fields_ = [("n", C.c_int64), ("rowptr", C.c_void_p), ("colidx", C.c_void_p), ("val", C.c_void_p)]


class nsp_opts(C.Structure):
    _fields_ = [("device", C.c_int), ("stream", C.c_void_p), ("nranks", C.c_int), ("rank", C.c_int),
                ("nccl_id", C.c_void_p), ("bcg_precond", C.c_int), ("factor_gamma", C.c_int),
                ("orth_tau", C.c_double), ("nys_eps_rel", C.c_double), ("scratch_bytes", C.c_size_t),
                ("verbose", C.c_int), ("local_group", C.c_void_p), ("apply_kernel", C.c_int),
                ("nys_power", C.c_int), ("nys_form", C.c_int), ("ag_order", C.c_int),
                ("ag_solver", C.c_int)]


class nsp_report(C.Structure):
    _fields_ = [("iters", C.c_int), ("converged", C.c_int), ("status", C.c_int), ("relres", C.c_double),
                ("hist", C.c_void_p), ("hist_cap", C.c_int), ("widths", C.c_void_p), ("widths_cap", C.c_int),
                ("bad_block", C.c_int), ("bad_pivot", C.c_longlong), ("rank", C.c_int), ("fallbacks", C.c_int),
                ("t_ms", C.c_double * 8)]


class NspError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{NSP_STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load_library(path: str = LIB_PATH):
    """Load libnsp.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} not built: run `python -m paper_2101_12164_b200.build`")
    lib = C.CDLL(path)
    P, I64, I, D = C.c_void_p, C.c_int64, C.c_int, C.c_double
    lib.nsp_default_opts.argtypes = [P]
    lib.nsp_default_opts.restype = None
    lib.nsp_setup.argtypes = [P, P, I, P, P, P]
    lib.nsp_dims.argtypes = [P, P, P, P, P]
    lib.nsp_gamma_index.argtypes = [P, P]
    lib.nsp_workspace_bytes.argtypes = [P, I, P]
    lib.nsp_stats.argtypes = [P, P]
    lib.nsp_ozaki_stats.argtypes = [P, P]
    lib.nsp_schur_apply.argtypes = [P, P, P, I, P]
    lib.nsp_kgamma_apply.argtypes = [P, P, P, I, P]
    lib.nsp_block_cg.argtypes = [P, P, P, I, D, I, P, P]
    lib.nsp_nystrom.argtypes = [P, I, I, C.c_uint64, P, D, I, P, P]
    lib.nsp_nystrom_sigma.argtypes = [P, P, P]
    lib.nsp_precond_apply.argtypes = [P, I, P, P, I, P]
    lib.nsp_pcg.argtypes = [P, P, P, D, I, I, P, P]
    lib.nsp_last_error.argtypes = [P]
    lib.nsp_last_error.restype = C.c_char_p
    lib.nsp_gamma_apply.argtypes = [P, P, P, I]
    lib.nsp_profile.argtypes = [P, I]
    lib.nsp_profile_read.argtypes = [P, P, P]
    lib.nsp_shard_plan.argtypes = [P, P, I, I, I, P, P, P, P, P]
    lib.nsp_shard_info.argtypes = [P, P, P, P, P]
    lib.nsp_nccl_unique_id.argtypes = [P]
    lib.nsp_nccl_selftest.argtypes = [I, C.c_size_t, P]
    lib.nsp_local_group_create.argtypes = [I]
    lib.nsp_local_group_create.restype = C.c_void_p
    lib.nsp_local_group_destroy.argtypes = [P]
    lib.nsp_local_group_destroy.restype = None
    lib.nsp_kernel_launches.argtypes = []
    lib.nsp_kernel_launches.restype = C.c_longlong
    lib.nsp_destroy.argtypes = [P]
    lib.nsp_destroy.restype = None
    lib.nsp_set_bcg_precond.argtypes = [P, I]
    lib.nsp_path_counters.argtypes = [P, I]
    lib.nsp_dev_panel.argtypes = [P, P, P, P, I64, I, D, P, I, P]
    lib.nsp_dev_gram.argtypes = [P, P, P, I64, I, P, P, I, I, P]
    lib.nsp_dev_panel_gram.argtypes = [P, P, P, P, I64, D, I, P, P, P]
    lib.nsp_dev_philox_gaussian.argtypes = [P, I64, I, C.c_uint64, C.c_uint, I64, P]
    lib.nsp_dev_set_fused_pg.argtypes = [I]
    for f in EXPORTED:
        if f not in ("nsp_default_opts", "nsp_last_error", "nsp_destroy", "nsp_kernel_launches",
                     "nsp_local_group_create", "nsp_local_group_destroy"):
            getattr(lib, f).restype = C.c_int
    _lib = lib
    return lib


def _ptr(t) -> int:
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError("expected a contiguous CUDA float64 tensor")
    return t.data_ptr() or None


class Report(dict):
    pass


def _report(rep: nsp_report, hist, widths) -> Report:
    r = Report(iters=rep.iters, converged=bool(rep.converged), status=rep.status, relres=rep.relres,
               bad_block=rep.bad_block, bad_pivot=rep.bad_pivot, rank=rep.rank, fallbacks=rep.fallbacks,
               t_ms=list(rep.t_ms))
    n = rep.iters + 1
    if hist is not None:
        r["hist"] = list(hist[: min(n, len(hist))])
    if widths is not None:
        r["widths"] = list(widths[: min(rep.iters, len(widths))])
    return r


def kernel_launches() -> int:
    return int(load_library().nsp_kernel_launches())


def path_counters() -> dict:
    """Dispatch-path counters (NSP_PATH_*): {name: dispatches so far in this process}."""
    lib = load_library()
    n = lib.nsp_path_counters(None, 0)
    out = (C.c_longlong * n)()
    lib.nsp_path_counters(out, n)
    return {nm: int(out[i]) for i, nm in enumerate(PATHS)}


def _stream_ptr(stream):
    import torch
    return (stream or torch.cuda.current_stream()).cuda_stream


def dev_panel(Out, Cin, In, M, sgn, colsq=None, path=0, stream=None):
    """nsp_dev_panel: Out = Cin + sgn * In M (n x s, s in {64, 128}); colsq = column sums of squares."""
    lib = load_library()
    st = lib.nsp_dev_panel(_ptr(Out), None if Cin is None else _ptr(Cin), _ptr(In), _ptr(M), In.shape[0],
                           In.shape[1], sgn, None if colsq is None else _ptr(colsq), path, _stream_ptr(stream))
    if st != 0:
        raise NspError(st, "nsp_dev_panel failed")


def dev_panel_gram(Out, Cin, In, M, sgn, gmode, gram, colsq=None, stream=None):
    """nsp_dev_panel_gram: Out = Cin + sgn In M and gram = In^T Out (gmode 0) / Out^T Out (gmode 1)."""
    lib = load_library()
    st = lib.nsp_dev_panel_gram(_ptr(Out), None if Cin is None else _ptr(Cin), _ptr(In), _ptr(M), In.shape[0], sgn,
                                gmode, _ptr(gram), None if colsq is None else _ptr(colsq), _stream_ptr(stream))
    if st != 0:
        raise NspError(st, "nsp_dev_panel_gram failed")


def dev_philox_gaussian(out, seed, stream_id=0, row0=0, stream=None):
    """nsp_dev_philox_gaussian: the device Omega generator into out (rows x s)."""
    st = load_library().nsp_dev_philox_gaussian(_ptr(out), out.shape[0], out.shape[1], seed, stream_id, row0,
                                                _stream_ptr(stream))
    if st != 0:
        raise NspError(st, "nsp_dev_philox_gaussian failed")


def dev_set_fused_pg(mode: int):
    """nsp_dev_set_fused_pg: 0 production threshold, 1 force the fused panel + Gram pass, 2 never."""
    if load_library().nsp_dev_set_fused_pg(mode) != 0:
        raise NspError(-1, "nsp_dev_set_fused_pg: mode in {0, 1, 2}")


def dev_gram(Xa, Xb, out, Xb2=None, out2=None, lower_first=False, path=0, stream=None):
    """nsp_dev_gram: out = Xa^T Xb (and out2 = Xa^T Xb2)."""
    lib = load_library()
    st = lib.nsp_dev_gram(_ptr(Xa), _ptr(Xb), None if Xb2 is None else _ptr(Xb2), Xa.shape[0], Xa.shape[1],
                          _ptr(out), None if out2 is None else _ptr(out2), int(lower_first), path,
                          _stream_ptr(stream))
    if st != 0:
        raise NspError(st, "nsp_dev_gram failed")


def shard_plan(rowptr, colidx, val, part, K, nranks, rank):
    """Host-only shard plan (no device needed): dict(n_private, n_shared, gamma_local, blk0, nblk)."""
    lib = load_library()
    rp = np.ascontiguousarray(rowptr, dtype=np.int64)
    ci = np.ascontiguousarray(colidx, dtype=np.int32)
    va = np.ascontiguousarray(val, dtype=np.float64)
    pa = np.ascontiguousarray(part, dtype=np.int32)
    csr = nsp_csr(rp.size - 1, rp.ctypes.data, ci.ctypes.data, va.ctypes.data)
    npv, nsh, b0, nb = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
    st = lib.nsp_shard_plan(C.byref(csr), pa.ctypes.data, K, nranks, rank, C.byref(npv), C.byref(nsh), None,
                            C.byref(b0), C.byref(nb))
    if st != 0:
        raise NspError(st, "nsp_shard_plan failed")
    gl = np.empty(npv.value + nsh.value, dtype=np.int64)
    lib.nsp_shard_plan(C.byref(csr), pa.ctypes.data, K, nranks, rank, None, None, gl.ctypes.data, None, None)
    return dict(n_private=npv.value, n_shared=nsh.value, gamma_local=gl, blk0=b0.value, nblk=nb.value)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    st = load_library().nsp_nccl_unique_id(buf)
    if st != 0:
        raise NspError(st, "nsp_nccl_unique_id: libnccl.so.2 not loadable")
    return buf.raw


def nccl_selftest(device: int = 0, count: int = 1 << 20) -> float:
    """One-rank NCCL communicator: allreduce `count` fp64 values in place; returns the largest deviation."""
    err = C.c_double(-1.0)
    st = load_library().nsp_nccl_selftest(int(device), int(count), C.byref(err))
    if st != 0:
        raise NspError(st, "nsp_nccl_selftest")
    return err.value


class LocalGroup:
    """nranks host threads driving ranks on ONE device (testing the sharded path; no NCCL)."""

    def __init__(self, nranks):
        self.lib = load_library()
        self.handle = self.lib.nsp_local_group_create(nranks)
        if not self.handle:
            raise ValueError("nranks must be in [1, 16]")

    def close(self):
        if self.handle:
            self.lib.nsp_local_group_destroy(self.handle)
            self.handle = None


class Context:
    """nsp_ctx owner.  A: (rowptr int64, colidx int32, val float64) host arrays."""

    def __init__(self, rowptr, colidx, val, part, K, device=0, stream=None, bcg_precond=0,
                 factor_gamma=False, orth_tau=1e-14, nys_eps_rel=1e-12, nranks=1, rank=0,
                 nccl_id: bytes | None = None, scratch_bytes=0, local_group: "LocalGroup | None" = None,
                 apply_kernel=0, nys_power=0, nys_form=0, ag_order=0, ag_solver=0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("CUDA device required (no CPU fallback)")
        self.lib = load_library()
        self._rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
        self._colidx = np.ascontiguousarray(colidx, dtype=np.int32)
        self._val = np.ascontiguousarray(val, dtype=np.float64)
        self._part = np.ascontiguousarray(part, dtype=np.int32)
        csr = nsp_csr(self._rowptr.size - 1, self._rowptr.ctypes.data, self._colidx.ctypes.data,
                      self._val.ctypes.data)
        o = nsp_opts()
        self.lib.nsp_default_opts(C.byref(o))
        o.device = device
        if stream is None:
            stream = torch.cuda.current_stream(device).cuda_stream
        o.stream = stream
        o.nranks, o.rank = nranks, rank
        self._nccl_id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        o.nccl_id = C.addressof(self._nccl_id) if self._nccl_id is not None else None
        o.bcg_precond = bcg_precond
        o.factor_gamma = int(bool(factor_gamma or bcg_precond))
        o.orth_tau, o.nys_eps_rel, o.scratch_bytes = orth_tau, nys_eps_rel, scratch_bytes
        o.local_group = local_group.handle if local_group is not None else None
        o.apply_kernel = apply_kernel
        o.nys_power = nys_power
        o.nys_form = nys_form
        o.ag_order = ag_order
        o.ag_solver = ag_solver
        self.opts = o
        self.ctx = C.c_void_p()
        rep = nsp_report()
        st = self.lib.nsp_setup(C.byref(csr), self._part.ctypes.data, K, C.byref(o), C.byref(self.ctx),
                                C.byref(rep))
        self.setup_report = _report(rep, None, None)
        if st != 0:
            msg = self.lib.nsp_last_error(self.ctx).decode()
            self.close()
            raise NspError(st, msg)
        n, ng, ngl, kl = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int()
        self._check(self.lib.nsp_dims(self.ctx, C.byref(n), C.byref(ng), C.byref(ngl), C.byref(kl)))
        self.n, self.n_gamma, self.n_gamma_local, self.K_local = n.value, ng.value, ngl.value, kl.value
        npv, nsh, b0, nb = C.c_int64(), C.c_int64(), C.c_int(), C.c_int()
        self._check(self.lib.nsp_shard_info(self.ctx, C.byref(npv), C.byref(nsh), C.byref(b0), C.byref(nb)))
        self.n_private, self.n_shared, self.blk0 = npv.value, nsh.value, b0.value

    def _check(self, st):
        if st < 0:
            raise NspError(st, self.lib.nsp_last_error(self.ctx).decode())
        return st

    def gamma_index(self) -> np.ndarray:
        out = np.empty(self.n_gamma_local, dtype=np.int64)
        self._check(self.lib.nsp_gamma_index(self.ctx, out.ctypes.data))
        return out

    def stats(self) -> dict:
        out = np.zeros(12, dtype=np.int64)
        self._check(self.lib.nsp_stats(self.ctx, out.ctypes.data))
        keys = ["n_I", "n_boundary_layer", "l22_entries", "factor_tiles", "nnz_AG", "nnz_AGI", "max_b", "ag_bw",
                "sum_b2", "sum_b", "n_sub", "wvu_rows"]
        return dict(zip(keys, [int(x) for x in out]))

    def ozaki_stats(self) -> dict:
        out = np.zeros(3, dtype=np.int64)
        self._check(self.lib.nsp_ozaki_stats(self.ctx, out.ctypes.data))
        return {"slice_products_executed": int(out[0]), "slice_products_full": int(out[1]),
                "m_slice_bytes": int(out[2])}

    def workspace_bytes(self, s: int) -> int:
        b = C.c_size_t()
        self._check(self.lib.nsp_workspace_bytes(self.ctx, s, C.byref(b)))
        return b.value

    def schur_apply(self, X, Y, ws=None):
        s = X.shape[1]
        self._check(self.lib.nsp_schur_apply(self.ctx, _ptr(X), _ptr(Y), s, None if ws is None else ws.data_ptr()))

    def kgamma_apply(self, X, Y, ws=None):
        s = X.shape[1]
        self._check(self.lib.nsp_kgamma_apply(self.ctx, _ptr(X), _ptr(Y), s, None if ws is None else ws.data_ptr()))

    def profile(self, enable=True):
        self._check(self.lib.nsp_profile(self.ctx, int(enable)))

    def profile_read(self):
        ms, cnt = C.c_double(), C.c_longlong()
        self._check(self.lib.nsp_profile_read(self.ctx, C.byref(ms), C.byref(cnt)))
        return ms.value, cnt.value

    def set_bcg_precond(self, precond: int):
        """nsp_set_bcg_precond: 0 = M = I, 1 = M = A_G^{-1} (reading C2) for later block_cg calls."""
        self._check(self.lib.nsp_set_bcg_precond(self.ctx, int(precond)))

    def gamma_apply(self, X, Y):
        self._check(self.lib.nsp_gamma_apply(self.ctx, _ptr(X), _ptr(Y), X.shape[1]))

    def block_cg(self, B, X, tol, maxit, ws=None, hist_cap=None):
        s = B.shape[1]
        cap = maxit + 1 if hist_cap is None else hist_cap
        hist = (C.c_double * cap)()
        widths = (C.c_int * cap)()
        rep = nsp_report()
        rep.hist, rep.hist_cap = C.addressof(hist), cap
        rep.widths, rep.widths_cap = C.addressof(widths), cap
        st = self.lib.nsp_block_cg(self.ctx, _ptr(B), _ptr(X), s, tol, maxit,
                                   None if ws is None else ws.data_ptr(), C.byref(rep))
        self._check(st)
        return _report(rep, hist, widths)

    def nystrom(self, rank, oversample, Omega, tol_inner, maxit_inner, ws=None, seed=0):
        """nsp_nystrom; Omega None -> generated on the device from `seed` (reading C7)."""
        cap = maxit_inner + 1
        hist = (C.c_double * cap)()
        widths = (C.c_int * cap)()
        rep = nsp_report()
        rep.hist, rep.hist_cap = C.addressof(hist), cap
        rep.widths, rep.widths_cap = C.addressof(widths), cap
        st = self.lib.nsp_nystrom(self.ctx, rank, oversample, seed, None if Omega is None else _ptr(Omega),
                                  tol_inner, maxit_inner,
                                  None if ws is None else ws.data_ptr(), C.byref(rep))
        self._check(st)
        r = _report(rep, hist, widths)
        r["status_code"] = st
        return r

    def nystrom_sigma(self, cap=4096) -> np.ndarray:
        out = np.zeros(cap)
        r = C.c_int()
        self._check(self.lib.nsp_nystrom_sigma(self.ctx, out.ctypes.data, C.byref(r)))
        return out[: r.value]

    def precond_apply(self, which, X, Y, ws=None):
        self._check(self.lib.nsp_precond_apply(self.ctx, which, _ptr(X), _ptr(Y), X.shape[1],
                                               None if ws is None else ws.data_ptr()))

    def pcg(self, b, x, tol, maxit, precond=2, ws=None):
        cap = maxit + 1
        hist = (C.c_double * cap)()
        rep = nsp_report()
        rep.hist, rep.hist_cap = C.addressof(hist), cap
        st = self.lib.nsp_pcg(self.ctx, _ptr(b), _ptr(x), tol, maxit, precond,
                              None if ws is None else ws.data_ptr(), C.byref(rep))
        self._check(st)
        return _report(rep, hist, None)

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            self.lib.nsp_destroy(self.ctx)
        self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
