"""Banded last-mode sharding with halo exchange (band
property bspline.hpp:27-30, G chain design.cpp:104-116).

CPU: the host plan kg_halo_plan (which slices each rank owns, touches, sends
and receives) on the BASELINE factors, and a gloo world-3 run of the exchange
protocol the library drives with NCCL send/recv (S(x) boundary partials go to
the owning neighbour, updated x boundary slices come back) reproducing the
all-reduced maps on every owned slice.  GPU: the owned-slice FISTA path on a
one-rank NCCL communicator (KG_HALO=1) against the unsharded fit."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1510_03298_b200 import _lib
from paper_1510_03298_b200 import kronglm as K


def plan(X, world, rank):
    out = (C.c_int64 * 9)()
    Xf = np.asfortranarray(X, dtype=np.float64)
    st = _lib.load().kg_halo_plan(X.shape[0], X.shape[1], Xf.ctypes.data_as(C.POINTER(C.c_double)), world, rank, out)
    assert st == 0
    ok, olo, ohi, tlo, thi, llo, lhi, rlo, rhi = list(out)
    return dict(ok=ok, own=(olo, ohi), touch=(tlo, thi), L=(llo, lhi), R=(rlo, rhi))


def rows(n, world, r):
    return n * r // world, n * (r + 1) // world


@pytest.mark.parametrize("n,p", [(1024, 256), (365, 60), (500, 120), (4096, 256)])
def test_halo_plan_partitions_and_neighbour_overlap(n, p):
    X = K.bspline_design(np.linspace(0, 1, n), 4, p)
    for world in (2, 4, 8):
        P = [plan(X, world, r) for r in range(world)]
        assert all(q["ok"] == 1 for q in P)
        assert P[0]["own"][0] == 0 and P[-1]["own"][1] == p
        for r in range(world):
            lo, hi = rows(n, world, r)
            nz = np.nonzero(np.any(X[lo:hi] != 0, axis=0))[0]
            assert P[r]["touch"] == (nz[0], nz[-1] + 1)
            if r + 1 < world:
                assert P[r]["own"][1] == P[r + 1]["own"][0]                # owned ranges tile [0, p)
                assert P[r]["R"] == P[r + 1]["L"]                          # what r sends is what r+1 receives
                assert P[r]["touch"][1] <= P[r + 1]["own"][1]              # the halo stays in the neighbour
            assert P[r]["touch"][0] >= P[r]["own"][0]
            assert P[r]["R"][1] - P[r]["R"][0] <= 4                        # cubic B-splines: <= 3-4 slices
        assert P[0]["L"][0] == P[0]["L"][1] and P[-1]["R"][0] == P[-1]["R"][1]


def test_halo_plan_rejects_ranks_narrower_than_the_band():
    X = K.bspline_design(np.linspace(0, 1, 40), 4, 10)
    assert any(plan(X, 20, r)["ok"] == 0 for r in range(20))  # 2 grid rows per rank
    assert all(plan(X, 2, r)["ok"] == 1 for r in range(2))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, p, q = 90, 24, 5  # last-mode grid rows, coefficient slices, p1 p2 of the other modes
        X = K.bspline_design(np.linspace(0, 1, n), 4, p)
        rng = np.random.default_rng(3)
        U = rng.standard_normal((q, n))    # G input (n-space, last mode unfolded)
        x = rng.standard_normal((q, p))    # coefficients
        P = plan(X, world, rank)
        lo, hi = rows(n, world, rank)
        (olo, ohi), (llo, lhi), (rlo, rhi) = P["own"], P["L"], P["R"]
        # --- S(x) partial of this slab, boundary exchange, owned sum
        part = U[:, lo:hi] @ X[lo:hi, :]
        reqs = []
        if rhi > rlo:
            reqs.append(dist.isend(torch.tensor(part[:, rlo:rhi].copy()), rank + 1))
        got = part.copy()
        if lhi > llo:
            buf = torch.empty((q, lhi - llo), dtype=torch.float64)
            dist.recv(buf, rank - 1)
            got[:, llo:lhi] += buf.numpy()
        for r_ in reqs:
            r_.wait()
        full = U @ X
        err_g = float(np.max(np.abs(got[:, olo:ohi] - full[:, olo:ohi])))
        untouched = np.delete(part, np.arange(P["touch"][0], P["touch"][1]), axis=1)
        zero_outside = bool(np.all(untouched == 0.0))  # nothing of this slab outside its touched slices
        # --- x halo: owned slices only, send the left overlap, receive the right halo
        xl = np.full_like(x, np.nan)
        xl[:, olo:ohi] = x[:, olo:ohi]
        reqs = []
        if lhi > llo:
            reqs.append(dist.isend(torch.tensor(xl[:, llo:lhi].copy()), rank - 1))
        if rhi > rlo:
            buf = torch.empty((q, rhi - rlo), dtype=torch.float64)
            dist.recv(buf, rank + 1)
            xl[:, rlo:rhi] = buf.numpy()
        for r_ in reqs:
            r_.wait()
        t0, t1 = P["touch"]
        eta = xl[:, t0:t1] @ X[lo:hi, t0:t1].T      # this slab's H from touched slices only
        err_h = float(np.max(np.abs(eta - (x @ X.T)[:, lo:hi])))
        halo_bytes = 8 * q * ((rhi - rlo) + (lhi - llo))
        out[rank] = (P["ok"], err_g, err_h, zero_outside, halo_bytes, ohi - olo)
    finally:
        dist.destroy_process_group()


def test_halo_exchange_protocol_gloo_world3():
    world = 3
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    res = [out[r] for r in range(world)]
    assert all(r[0] == 1 for r in res)
    assert max(r[1] for r in res) <= 1e-12
    assert max(r[2] for r in res) <= 1e-12
    assert all(r[3] for r in res)
    assert sum(r[5] for r in res) == 24
    assert max(r[4] for r in res) < 8 * 5 * 24  # boundary slices only, not the p-vector


@pytest.mark.gpu
def test_halo_path_world1_matches_unsharded(monkeypatch):
    """KG_HALO=1 runs the owned-slice FISTA path (update on the owned slices,
    boundary exchanges, 4-scalar all-reduce, owned all-gather) on a one-rank
    NCCL communicator, where every slice is owned and the exchanges are empty."""
    from tests.test_gpu_parity import bspline_design, compare_paths
    from paper_1510_03298_b200 import configs

    monkeypatch.setenv("KG_HALO", "1")
    uid = K.nccl_unique_id()
    ctx = K.Context.sharded(0, 0, 1, uid)
    rng = np.random.default_rng(29)
    design = bspline_design((64, 64, 40), (16, 16, 12))
    B = np.zeros((16, 16, 12))
    m = rng.random(B.shape) < 0.1
    B[m] = rng.standard_normal(m.sum())
    eta = configs.tensor_h(design[0], B)
    y = rng.poisson(np.exp(np.log(20.0) / eta.max() * eta)).astype(float)
    D = K.Design(design, ctx)
    hp = (C.c_int64 * 9)()
    assert _lib.load().kg_design_halo(D.h, hp) == 0
    assert list(hp)[:3] == [1, 0, 12]
    kw = dict(n_lambda=6, lambda_min_ratio=1e-2)
    got = K.fit_path_resident(D, K.Observation(D, y), "poisson", **kw)
    want = K.fit_path(design, "poisson", y, **kw)
    res = {"lambdas": got.lambdas, "objectives": got.objectives, "truncated": got.truncated,
           "coefficients": [D.blocks(c) for c in got.coefs()], "outer_iters": got.outer_iters,
           "inner_iters": got.inner_iters}
    compare_paths(res, want)
    ctx.close()
