"""The product's last-mode sharded contexts in two processes.

Two ranks on one GPU, each a kg_ctx_create_sharded context of world 2 without
a communicator (local partials only: NCCL needs one GPU per rank), reduce
their partials with torch.distributed's gloo backend.  One full FISTA step of
the first Poisson outer iteration -- the slab's linear predictor, the weights
and working response, X^T W X theta, b = X^T W z, the gradient (S - b)/n,
the objective partial and the prox step -- must equal the same step computed
by an unsharded context on the whole array (1e-12 relative)."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N, P = (20, 16, 24), (6, 5, 8)


def _problem():
    from paper_1510_03298_b200 import configs
    from paper_1510_03298_b200 import kronglm as K
    rng = np.random.default_rng(7)
    design = [[K.bspline_design(np.linspace(0, 1, n), 4, p) for n, p in zip(N, P)]]
    B = np.zeros(P)
    m = rng.random(P) < 0.2
    B[m] = rng.standard_normal(int(m.sum()))
    eta = configs.tensor_h(design[0], B)
    y = np.asfortranarray(rng.poisson(np.exp(np.log(20.0) / eta.max() * eta)).astype(float))
    theta = [np.asfortranarray(0.05 * rng.standard_normal(P))]
    return design, y, theta


def _step(K, D, y, theta):
    """Local pieces of one FISTA gradient step on this context's slab."""
    eta = K.h_map(D, theta)
    mu = np.exp(np.clip(eta, -30, 30))  # glm_weights / working_response (family.cpp:198-261)
    v = np.asfortranarray(np.maximum(mu, 1e-10))
    z = np.asfortranarray((y - mu) / np.maximum(mu, 1e-10) + eta)
    S = np.concatenate([b.ravel(order="F") for b in K.xtwx_apply(D, v, theta)])
    b = np.concatenate([c.ravel(order="F") for c in K.g_map(D, np.asfortranarray(v * z))])
    ss = float(np.sum(v * (eta - z) ** 2))
    return eta, S, b, ss


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_1510_03298_b200 import kronglm as K
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        design, y, theta = _problem()
        ctx = K.Context.sharded(0, rank, world, None)
        D = K.Design(design, ctx)
        lo, hi = K.shard_rows(N[-1], rank, world)
        eta, S, b, ss = _step(K, D, np.asfortranarray(y[..., lo:hi]), theta)
        t = torch.tensor(np.concatenate([S, b, [ss]]), dtype=torch.float64)
        dist.all_reduce(t)
        out[rank] = {"eta": eta, "sum": t.numpy().copy(), "lohi": (lo, hi)}
        D.close()
        ctx.close()
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_sharded_gradient_step_matches_unsharded():
    import torch.multiprocessing as mp
    from paper_1510_03298_b200 import kronglm as K
    world = 2
    port = _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    design, y, theta = _problem()
    D = K.Design(design)
    eta, S, b, ss = _step(K, D, y, theta)
    p = S.size
    for r in range(world):  # each slab's linear predictor is the full one's slab
        lo, hi = res[r]["lohi"]
        np.testing.assert_allclose(res[r]["eta"], eta[..., lo:hi], rtol=0, atol=1e-12 * np.max(np.abs(eta)))
    tot = res[0]["sum"]
    np.testing.assert_array_equal(tot, res[1]["sum"])  # identical replicated state on both ranks
    S2, b2, ss2 = tot[:p], tot[p:2 * p], tot[2 * p]
    assert np.max(np.abs(S2 - S)) <= 1e-12 * np.max(np.abs(S))
    assert np.max(np.abs(b2 - b)) <= 1e-12 * np.max(np.abs(b))
    assert abs(ss2 - ss) <= 1e-12 * abs(ss)
    # the FISTA step from the summed partials (inner.cpp:163-186 with omega = 0)
    n = float(np.prod(N))
    lip = float(np.max(np.exp(np.clip(eta, -30, 30)))) * np.prod([D.spectral(0, j) for j in range(3)]) / n
    th = np.concatenate([t.ravel(order="F") for t in theta])
    lam = 1e-3

    def prox_step(Sv, bv):
        g = (Sv - bv) / n
        u = th - g / lip
        return np.sign(u) * np.maximum(np.abs(u) - lam / lip, 0.0)

    x_sh, x_full = prox_step(S2, b2), prox_step(S, b)
    assert np.array_equal(x_sh != 0, x_full != 0)
    assert np.max(np.abs(x_sh - x_full)) <= 1e-12 * max(np.max(np.abs(x_full)), 1e-300)
