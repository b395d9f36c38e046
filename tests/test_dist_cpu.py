"""CPU coverage of the sharded (N > 1) path: the library's host-only shard plan
(nsp_shard_plan) and, on world_size-2/4 gloo process groups, the distributed S_G apply and Gram rule
the CUDA path implements - each rank applies only its own blocks and private rows, the shared
rows' partials are summed by an allreduce, the shared x shared A_G term is added after it, and
Grams count the private rows of every rank plus the shared rows once (rank 0).  The per-rank
arithmetic here is the oracle's (scipy block solves); the plan is the product library's."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
from nsp_inputs import philox
from nsp_inputs import problems as P
from paper_2101_12164_b200 import nsp


def _plan(pr, G, r):
    return nsp.shard_plan(pr.A.rowptr, pr.A.colidx, pr.A.val, pr.part, pr.K, G, r)


@pytest.mark.parametrize("name", ["cfg1", "cfg2s", "cfg5s", "cfg4s"])
@pytest.mark.parametrize("G", [1, 2, 4, 8])
def test_shard_plan_invariants(name, G):
    pr = P.make(name)
    if G > pr.K:
        pytest.skip("more ranks than blocks")
    A = pr.A.to_scipy().tocsr()
    gamma = np.flatnonzero(pr.part < 0)
    plans = [_plan(pr, G, r) for r in range(G)]
    shared = [tuple(p["gamma_local"][p["n_private"]:]) for p in plans]
    assert all(sh == shared[0] for sh in shared)                     # replicated shared rows
    priv = [set(p["gamma_local"][: p["n_private"]]) for p in plans]
    allp = set().union(*priv)
    assert sum(len(x) for x in priv) == len(allp)                    # private sets disjoint
    assert allp | set(shared[0]) == set(gamma) and not (allp & set(shared[0]))
    # contiguous block ranges covering [0, K)
    starts = [p["blk0"] for p in plans]
    assert starts[0] == 0 and all(plans[r]["blk0"] + plans[r]["nblk"] == (plans[r + 1]["blk0"] if r + 1 < G else pr.K)
                                  for r in range(G))
    for r, p in enumerate(plans):
        loc = set(p["gamma_local"])
        mine = (pr.part >= p["blk0"]) & (pr.part < p["blk0"] + p["nblk"])
        # every Gamma neighbour of a local block is a local Gamma row
        rows = np.flatnonzero(mine)
        nb = A[rows].tocoo()
        gcols = nb.col[pr.part[nb.col] < 0]
        assert set(gcols.tolist()) <= loc
        # a private row only touches own blocks and local Gamma rows
        pv = np.array(sorted(priv[r]), dtype=np.int64)
        if pv.size:
            sub = A[pv].tocoo()
            cols = sub.col
            blk = pr.part[cols]
            assert np.all((blk < 0) | ((blk >= p["blk0"]) & (blk < p["blk0"] + p["nblk"])))
            assert set(cols[blk < 0].tolist()) <= loc
        # ascending original ids within each group
        assert np.all(np.diff(p["gamma_local"][: p["n_private"]]) > 0)
        assert np.all(np.diff(p["gamma_local"][p["n_private"]:]) > 0)
    if G == 1:
        assert np.array_equal(plans[0]["gamma_local"], gamma) and plans[0]["n_private"] == gamma.size


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, G, name, port, s, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=G)
    try:
        pr = P.make(name)
        d = O.dbbd(pr.A.to_scipy(), pr.part, pr.K)
        S = O.SchurOracle(d)
        p = _plan(pr, G, rank)
        gl = p["gamma_local"]
        npv = p["n_private"]
        pos = np.searchsorted(d.gamma, gl)                      # local row -> global Gamma position
        assert np.array_equal(d.gamma[pos], gl)
        X = philox.gaussian_block(3, 9, d.n_gamma, s)
        Xl = X[pos]                                             # this rank's rows only
        AGl = d.A_G[pos][:, pos].tocsr()
        Y = np.zeros((gl.size, s))
        # A_G term: private rows all local columns; shared rows only this rank's private columns
        Y[:npv] = AGl[:npv] @ Xl
        Y[npv:] = AGl[npv:, :npv] @ Xl[:npv]
        # K_G term of this rank's blocks only (A_IG restricted to local Gamma columns)
        for j in range(p["blk0"], p["blk0"] + p["nblk"]):
            AIG = d.A_IG[j][:, pos]
            assert AIG.nnz == d.A_IG[j].nnz                     # block j touches local rows only
            U = S.solve_AI_block(j, AIG @ Xl)
            Y -= AIG.T @ U
        t = torch.from_numpy(np.ascontiguousarray(Y[npv:]))
        dist.all_reduce(t)                                      # one allreduce of the shared partials
        Y[npv:] = t.numpy() + AGl[npv:, npv:] @ Xl[npv:]        # + shared x shared A_G term
        ref = S.apply(X)[pos]
        err_apply = float(np.linalg.norm(Y - ref) / np.linalg.norm(ref))
        # shared rows bitwise identical across ranks
        sh = torch.from_numpy(np.ascontiguousarray(Y[npv:]))
        sh0 = sh.clone()
        dist.broadcast(sh0, 0)
        same = bool(torch.equal(sh, sh0))
        # Gram rule: private rows of every rank + shared rows once (rank 0)
        ng = gl.size if rank == 0 else npv
        Gm = torch.from_numpy(np.ascontiguousarray(Xl[:ng].T @ Y[:ng]))
        dist.all_reduce(Gm)
        err_gram = float(np.linalg.norm(Gm.numpy() - X.T @ S.apply(X)) / np.linalg.norm(X.T @ S.apply(X)))
        out[rank] = (err_apply, same, err_gram)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,G", [("cfg2s", 2), ("cfg5s", 2), ("cfg4s", 2), ("cfg5s", 4)])
def test_distributed_apply_and_gram_gloo(name, G):
    import torch.multiprocessing as mp
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(G, name, _free_port(), 16, out), nprocs=G, join=True)
    for r in range(G):
        err_apply, same, err_gram = out[r]
        assert err_apply <= 1e-12, (r, err_apply)
        assert same
        assert err_gram <= 1e-12, (r, err_gram)
