"""Kernel-level parity of the block-CG building blocks (rows a6, a8, a10, a11) that the bench's
s = 128 path dispatches - the one-wave row-range panel (k_panel_rows, n >= 64 x SMs) and the
symmetric / [D | E] Gram variants - against the plain definitions Out = Cin + sgn In M and
out = Xa^T Xb computed in fp64 by numpy (the same contraction, a library primitive).  Shapes straddle
the dispatch threshold and end on ragged tails; the path counters prove which kernel ran."""
import numpy as np
import pytest
import torch

from paper_2101_12164_b200 import nsp
from tests.gpu_util import block

pytestmark = pytest.mark.gpu


def _nsm():
    return torch.cuda.get_device_properties(0).multi_processor_count


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _shapes():
    n0 = 64 * _nsm()
    return [(n0 - 1, 128), (n0, 128), (14287, 128), (20001, 128), (3687, 64), (14287, 64), (1, 128), (0, 128)]


@pytest.mark.parametrize("idx", range(8))
@pytest.mark.parametrize("path", [0, 1])
def test_panel_matches_definition(idx, path):
    n, s = _shapes()[idx]
    In = block(max(n, 1), s, seed=11)[:n]
    M = block(s, s, seed=12)
    Cin = block(max(n, 1), s, seed=13)[:n]
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    Out = torch.empty(n, s, dtype=torch.float64, device="cuda")
    cs = torch.empty(s, dtype=torch.float64, device="cuda")
    before = nsp.path_counters()
    nsp.dev_panel(Out, d(Cin), d(In), d(M), -1.0, colsq=cs, path=path)
    after = nsp.path_counters()
    ref = Cin - In @ M
    if n:
        assert _rel(Out.cpu().numpy(), ref) <= 1e-13
    assert _rel(cs.cpu().numpy(), (ref * ref).sum(axis=0)) <= 1e-13 if n else float(cs.abs().max()) == 0.0
    rows = path == 0 and s == 128 and n >= 64 * _nsm()
    if n:   # (an empty block returns before any dispatch)
        assert after["panel_rows"] - before["panel_rows"] == (1 if rows else 0)
        assert after["panel_tiles"] - before["panel_tiles"] == (0 if rows else 1)
    # in place (Out aliases Cin: R -= Q alpha) and without Cin (P = W T)
    R = d(Cin)
    nsp.dev_panel(R, R, d(In), d(M), -1.0, path=path)
    assert n == 0 or _rel(R.cpu().numpy(), ref) <= 1e-13
    nsp.dev_panel(Out, None, d(In), d(M), 1.0, path=path)
    assert n == 0 or _rel(Out.cpu().numpy(), In @ M) <= 1e-13


@pytest.mark.parametrize("idx", range(8))
@pytest.mark.parametrize("path", [0, 1])
def test_gram_matches_definition(idx, path):
    n, s = _shapes()[idx]
    Xa = block(n, s, seed=21)
    Xb = block(n, s, seed=22)
    Xc = block(n, s, seed=23)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    out = torch.empty(s, s, dtype=torch.float64, device="cuda")
    out2 = torch.empty(s, s, dtype=torch.float64, device="cuda")
    A = d(Xa)
    before = nsp.path_counters()
    nsp.dev_gram(A, A, out, path=path)                      # W^T W
    after = nsp.path_counters()
    G = out.cpu().numpy()
    if n == 0:
        assert not G.any()
        return
    assert _rel(G, Xa.T @ Xa) <= 1e-13
    assert np.array_equal(G, G.T)                            # the symmetric path mirrors exactly
    sym = path == 0 and s > 64
    if n:
        assert after["gram_sym"] - before["gram_sym"] == (1 if sym else 0)
    nsp.dev_gram(A, d(Xb), out, Xb2=d(Xc), out2=out2, lower_first=True, path=path)   # [D | E]
    after2 = nsp.path_counters()
    D, E = out.cpu().numpy(), out2.cpu().numpy()
    ref = Xa.T @ Xb
    assert _rel(np.tril(D), np.tril(ref)) <= 1e-13
    assert _rel(E, Xa.T @ Xc) <= 1e-13
    assert after2["gram_de"] - after["gram_de"] == (1 if sym else 0)
    nsp.dev_gram(A, d(Xb), out, path=path)                  # Q^T R (full tiles)
    assert _rel(out.cpu().numpy(), ref) <= 1e-13


def test_gram_deterministic():
    """Reading C17: fixed-order reductions - repeated Grams are bitwise identical."""
    n, s = 14287, 128
    A = torch.from_numpy(block(n, s, seed=31)).cuda()
    o1 = torch.empty(s, s, dtype=torch.float64, device="cuda")
    o2 = torch.empty_like(o1)
    nsp.dev_gram(A, A, o1)
    nsp.dev_gram(A, A, o2)
    assert torch.equal(o1, o2)


@pytest.mark.parametrize("n", ["nsm", 14287, 20001, 200003])
@pytest.mark.parametrize("gmode", [0, 1])
def test_fused_panel_gram(n, gmode):
    """The fused pass against its definition: Out = Cin + sgn In M, gram = In^T Out / Out^T Out."""
    n = 64 * _nsm() if n == "nsm" else n
    s = 128
    In = block(n, s, seed=41)
    M = block(s, s, seed=42) * 0.1
    Cin = block(n, s, seed=43)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    Out = torch.empty(n, s, dtype=torch.float64, device="cuda")
    G = torch.empty(s, s, dtype=torch.float64, device="cuda")
    cs = torch.empty(s, dtype=torch.float64, device="cuda")
    sgn = -1.0 if gmode == 0 else 1.0
    before = nsp.path_counters()
    nsp.dev_panel_gram(Out, d(Cin), d(In), d(M), sgn, gmode, G, colsq=cs)
    assert nsp.path_counters()["panel_gram"] == before["panel_gram"] + 1
    ref = Cin + sgn * (In @ M)
    assert _rel(Out.cpu().numpy(), ref) <= 1e-13
    Gr = (In.T @ ref) if gmode == 0 else (ref.T @ ref)
    Gg = G.cpu().numpy()
    assert _rel(Gg, Gr) <= 1e-13
    if gmode == 1:
        assert np.array_equal(Gg, Gg.T)
    assert _rel(cs.cpu().numpy(), (ref * ref).sum(axis=0)) <= 1e-13
    # in place (Out aliases Cin, as R -= Q alpha)
    R = d(Cin)
    nsp.dev_panel_gram(R, R, d(In), d(M), sgn, gmode, G)
    assert _rel(R.cpu().numpy(), ref) <= 1e-13
    assert _rel(G.cpu().numpy(), Gr) <= 1e-13


@pytest.mark.parametrize("seed,stream_id,row0,rows,s", [(0, 0, 0, 4096, 30), (7, 9, 123457, 1000, 128),
                                                        (2**40 + 3, 1, 10**9, 64, 1)])
def test_device_philox_matches_host_generator(seed, stream_id, row0, rows, s):
    """Reading C7: the device Omega generator equals nsp_inputs.philox (counter (e, stream, 0), key seed,
    Box-Muller cosine branch) up to the last-ulp rounding of log / cos (<= 4 ulp); row0 = 0 is exactly
    philox.gaussian_block."""
    from nsp_inputs import philox
    out = torch.empty(rows, s, dtype=torch.float64, device="cuda")
    nsp.dev_philox_gaussian(out, seed, stream_id, row0)
    u1, u2 = philox._uniform_pair(philox._raw(seed, stream_id, row0 * s, rows * s))
    ref = (np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)).reshape(rows, s)
    if row0 == 0:
        assert np.array_equal(ref, philox.gaussian_block(seed, stream_id, rows, s))
    got = out.cpu().numpy()
    assert np.all(np.abs(got - ref) <= 4 * np.spacing(np.abs(ref)) + 1e-300)
