"""World-size-2 gloo test of the last-mode sharding decomposition (CPU): slab
H maps and all-reduced slab G maps / scalar partials reproduce the
single-device maps, lambda_max and the FISTA gradient."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from tests import slab_split as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _design():
    rng = np.random.default_rng(8)
    n, p = (12, 9, 10), (5, 4, 6)
    X = [O.bspline_design(np.linspace(0, 1, k), 4, q) for k, q in zip(n, p)]
    th = rng.standard_normal(p)
    y = rng.standard_normal(n)
    v = rng.uniform(0.5, 2.0, n)
    return [X], [th], y, v


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
        design, th, y, v = _design()
        n = y.shape
        sl = S.slab(n, rank, world)
        dl = S.shard_design(design, sl)
        # H is local: the slab of the full map
        eta_l = O.h_map(dl, th)
        full = O.h_map(design, th)
        ok_h = np.array_equal(eta_l, S.shard_array(full, sl))
        # G: all-reduced slab partials
        u_l = S.shard_array(y, sl)
        g_l = torch.tensor(np.concatenate([b.ravel(order="F") for b in O.g_map(dl, u_l)]))
        dist.all_reduce(g_l)
        g_full = np.concatenate([b.ravel(order="F") for b in O.g_map(design, y)])
        err_g = float(np.max(np.abs(g_l.numpy() - g_full)))
        # lambda_max: all-reduce of the G partial, then max |.| / n_global
        lmax = float(np.max(np.abs(g_l.numpy()))) / float(np.prod(n))
        err_l = abs(lmax - O.lambda_max(design, "gaussian", y))
        # gradient of h at theta: (X^T V X th - X^T V y) / n via slab partials
        v_l = S.shard_array(v, sl)
        s_l = torch.tensor(np.concatenate([b.ravel(order="F") for b in O.xtwx_apply(dl, v_l, th)]))
        b_l = torch.tensor(np.concatenate([b.ravel(order="F") for b in O.g_map(dl, v_l * u_l)]))
        ss_l = torch.tensor([float(np.sum(v_l * (eta_l - u_l) ** 2))], dtype=torch.float64)
        vmax = torch.tensor([float(v_l.max())], dtype=torch.float64)
        for t in (s_l, b_l, ss_l):
            dist.all_reduce(t)
        dist.all_reduce(vmax, op=dist.ReduceOp.MAX)
        grad = (s_l.numpy() - b_l.numpy()) / float(np.prod(n))
        s_f = np.concatenate([b.ravel(order="F") for b in O.xtwx_apply(design, v, th)])
        b_f = np.concatenate([b.ravel(order="F") for b in O.g_map(design, v * y)])
        err_grad = float(np.max(np.abs(grad - (s_f - b_f) / float(np.prod(n)))))
        ss_f = float(np.sum(v * (full - y) ** 2))
        err_ss = abs(float(ss_l.item()) - ss_f) / ss_f
        out[rank] = (ok_h, err_g, err_l, err_grad, err_ss, float(vmax.item()) == float(v.max()), sl.cell_base)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_last_mode_sharding_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for rank in range(world):
        ok_h, err_g, err_l, err_grad, err_ss, ok_vmax, base = out[rank]
        assert ok_h
        assert err_g <= 1e-12 and err_l <= 1e-14 and err_grad <= 1e-13 and err_ss <= 1e-13
        assert ok_vmax
    assert out[0][6] == 0 and out[1][6] == 12 * 9 * 5


def test_slab_plan_partitions_cells():
    for ext, world in (((4, 3, 10), 3), ((7,), 2), ((5, 8), 8)):
        slabs = [S.slab(ext, r, world) for r in range(world)]
        assert slabs[0].lo == 0 and slabs[-1].hi == ext[-1]
        assert sum(s.n_local for s in slabs) == int(np.prod(ext))
        for a, b in zip(slabs, slabs[1:]):
            assert a.hi == b.lo and a.cell_base + a.n_local == b.cell_base
    with pytest.raises(ValueError):
        S.slab((4, 3), 0, 4)
