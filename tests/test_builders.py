"""Input builders in front of the fit path: bin_scatter
(bspline.cpp:106-153) and the device bspline_design (bspline.cpp:64-104).

CPU: the oracle restatement against the reference's known answers
(proj/tests/test_bspline.cpp:122-160).  GPU: the CUDA builders bit-exact
against the oracle (counts are integers; the design uses explicitly rounded
FP64), on both kernel paths (shared-memory privatised and global atomics)."""
import numpy as np
import pytest

from oracle import oracle as O


def _naive2(pts, bins):  # test_bspline.cpp:141-152
    out = np.zeros((bins, bins))
    dropped = 0
    for x, y in pts:
        if x < 0 or x > 1 or y < 0 or y > 1:
            dropped += 1
            continue
        out[min(int(x * bins), bins - 1), min(int(y * bins), bins - 1)] += 1
    return out, dropped


# ------------------------------------------------------------ oracle pins (CPU)
def test_oracle_bin_scatter_corner_and_boundary():
    counts, dropped = O.bin_scatter([[0.0, 0.0], [1.0, 2.0], [0.499, 1.999]], [(0, 1), (0, 2)], [2, 4])
    assert dropped == 0
    assert counts.shape == (2, 4)
    assert counts[0, 0] == 1 and counts[1, 3] == 1 and counts[0, 3] == 1 and counts.sum() == 3


def test_oracle_bin_scatter_drops_out_of_bounds():
    counts, dropped = O.bin_scatter([[-0.1, 0.5], [0.5, 2.5], [0.5, 0.5]], [(0, 1), (0, 2)], [2, 2])
    assert dropped == 2 and counts.sum() == 1


def test_oracle_bin_scatter_matches_naive_binner():
    rng = np.random.default_rng(82)
    pts = rng.uniform(-0.1, 1.1, size=(10000, 2))
    counts, dropped = O.bin_scatter(pts, [(0, 1), (0, 1)], [4, 4])
    want, wd = _naive2(pts, 4)
    assert dropped == wd and counts.sum() == 10000 - wd
    assert np.array_equal(counts, want)


def test_oracle_bin_scatter_errors():
    with pytest.raises(ValueError, match="need at least one bin"):
        O.bin_scatter([[0.5]], [(0, 1)], [0])
    with pytest.raises(ValueError, match="degenerate bounds"):
        O.bin_scatter([[0.5]], [(1, 1)], [2])
    with pytest.raises(ValueError, match="agree on the dimension"):
        O.bin_scatter([[0.5]], [(0, 1), (0, 1)], [2])


# ------------------------------------------------------------ device (GPU)
def _edge_points(rng, n, d, bins, lo, hi):
    """Uniform points spilling past the bounds, plus points exactly on the
    bounds and on interior bin edges, and non-finite coordinates."""
    pts = rng.uniform(-0.1, 1.1, size=(n, d)) * (hi - lo) + lo
    k = max(n // 10, 1)
    for j in range(d):
        edge = lo[j] + (hi[j] - lo[j]) / bins[j] * rng.integers(0, bins[j] + 1, size=k)
        pts[rng.integers(0, n, size=k), j] = edge
    pts[rng.integers(0, n, size=3), rng.integers(0, d, size=3)] = [np.nan, np.inf, -np.inf]
    return pts


CASES = [  # (d, bins, npts): shared-memory counters when they fit (~37K cells at d=3) and npts >= 8 cells
    (1, [7], 20000),
    (2, [4, 4], 10000),
    (2, [1, 3], 5000),
    (3, [10, 20, 30], 100000),
    (3, [64, 64, 16], 100000),   # 65536 cells: global-atomic path
    (4, [3, 4, 5, 6], 50000),
    (5, [2, 3, 2, 3, 2], 20000),  # generic-d kernel
    (8, [2, 2, 2, 2, 2, 2, 2, 3], 30000),
    (2, [300, 300], 1000),       # few points per cell: global path
]


@pytest.mark.gpu
@pytest.mark.parametrize("d,bins,npts", CASES)
def test_bin_scatter_matches_oracle(d, bins, npts):
    from paper_1510_03298_b200 import kronglm as K
    rng = np.random.default_rng(1000 + d * 7 + npts % 97)
    lo = rng.uniform(-5, 5, size=d)
    hi = lo + rng.uniform(0.5, 10, size=d)
    pts = _edge_points(rng, npts, d, bins, lo, hi)
    bounds = list(zip(lo, hi))
    want, wd = O.bin_scatter(pts, bounds, bins)
    got = K.bin_scatter(pts, bounds, bins)
    assert got.dropped == wd
    assert got.counts.shape == tuple(bins)
    assert np.array_equal(got.counts, want)


@pytest.mark.gpu
def test_bin_scatter_unaligned_device_points():
    """A device point array that is not 16-byte aligned takes the direct-load
    kernel; ragged tile tails on both kernels."""
    import torch
    from paper_1510_03298_b200 import kronglm as K
    rng = np.random.default_rng(77)
    for npts, bins in ((100_001, [5, 6, 7]), (3_333, [50, 50, 50])):
        flat = torch.from_numpy(rng.uniform(-0.05, 1.05, size=3 * npts + 1)).cuda()
        for off in (0, 1):
            pts = flat[off:off + 3 * npts].view(npts, 3)
            out = torch.empty(int(np.prod(bins)), device="cuda", dtype=torch.float64)
            r = K.bin_scatter(pts, [(0, 1)] * 3, bins, out=out)
            want, wd = O.bin_scatter(pts.cpu().numpy(), [(0, 1)] * 3, bins)
            assert r.dropped == wd
            assert np.array_equal(out.cpu().numpy(), want.reshape(-1, order="F"))


@pytest.mark.gpu
def test_bin_scatter_reference_known_answers():
    from paper_1510_03298_b200 import kronglm as K
    r = K.bin_scatter([[0.0, 0.0], [1.0, 2.0], [0.499, 1.999]], [(0, 1), (0, 2)], [2, 4])
    assert r.dropped == 0 and r.counts[0, 0] == 1 and r.counts[1, 3] == 1 and r.counts[0, 3] == 1
    r = K.bin_scatter([[-0.1, 0.5], [0.5, 2.5], [0.5, 0.5]], [(0, 1), (0, 2)], [2, 2])
    assert r.dropped == 2 and r.counts.sum() == 1
    rng = np.random.default_rng(82)
    pts = rng.uniform(-0.1, 1.1, size=(10000, 2))
    r = K.bin_scatter(pts, [(0, 1), (0, 1)], [4, 4])
    want, wd = _naive2(pts, 4)
    assert r.dropped == wd and np.array_equal(r.counts, want)


@pytest.mark.gpu
def test_bin_scatter_empty_skewed_and_errors():
    from paper_1510_03298_b200 import kronglm as K
    r = K.bin_scatter(np.zeros((0, 3)), [(0, 1)] * 3, [2, 3, 4])
    assert r.dropped == 0 and r.counts.shape == (2, 3, 4) and not r.counts.any()
    # every point in one cell: warp-aggregated shared-memory counters
    pts = np.full((1_000_003, 2), 0.25)
    r = K.bin_scatter(pts, [(0, 1), (0, 1)], [8, 8])
    assert r.counts[2, 2] == 1_000_003 and r.counts.sum() == 1_000_003
    with pytest.raises(ValueError, match="need at least one bin"):
        K.bin_scatter([[0.5]], [(0, 1)], [0])
    with pytest.raises(ValueError, match="degenerate bounds"):
        K.bin_scatter([[0.5]], [(1, 1)], [2])
    with pytest.raises(ValueError, match="agree on the dimension"):
        K.bin_scatter([[0.5]], [(0, 1), (0, 1)], [2])
    with pytest.raises(ValueError, match="point arity"):
        K.bin_scatter(np.zeros((4, 3)), [(0, 1)] * 2, [2, 2])


@pytest.mark.gpu
def test_bin_scatter_full_size_device_resident_feeds_observation():
    """BASELINE-scale count arrays (C2's 100x100x120 grid) from 20M device
    points: counts + dropped == npts, equal to the oracle on the same points,
    and the device counts feed Observation without a host round trip (the
    Poisson fit equals the one on host-uploaded counts)."""
    import torch
    from paper_1510_03298_b200 import kronglm as K
    g = torch.Generator(device="cuda").manual_seed(5)
    npts, bins = 20_000_000, [100, 100, 120]
    pts = torch.rand((npts, 3), generator=g, device="cuda", dtype=torch.float64) * 1.2 - 0.1
    out = torch.empty(int(np.prod(bins)), device="cuda", dtype=torch.float64)
    r = K.bin_scatter(pts, [(0, 1)] * 3, bins, out=out)
    torch.cuda.synchronize()
    host = out.cpu().numpy()
    assert host.sum() + r.dropped == npts
    want, wd = O.bin_scatter(pts.cpu().numpy(), [(0, 1)] * 3, bins)
    assert r.dropped == wd and np.array_equal(host, want.reshape(-1, order="F"))
    # counts -> Observation on the device; a small design keeps the fit quick
    small = [20, 20, 24]
    out_s = torch.empty(int(np.prod(small)), device="cuda", dtype=torch.float64)
    K.bin_scatter(pts[:2_000_000].contiguous(), [(0, 1)] * 3, small, out=out_s)
    comps = [[K.bspline_design(np.arange(1.0, n + 1.0), 4, K.default_basis_count(n, 4)) for n in small]]
    D = K.Design(comps)
    res_dev = K.fit_path_resident(D, K.Observation(D, out_s), "poisson", n_lambda=4)
    y_host = out_s.cpu().numpy().reshape(small, order="F")
    res_host = K.fit_path_resident(D, K.Observation(D, y_host), "poisson", n_lambda=4)
    assert res_dev.lambdas == res_host.lambdas
    assert np.array_equal(res_dev.coefs(), res_host.coefs())


@pytest.mark.gpu
@pytest.mark.parametrize("order", [1, 2, 3, 4, 5])
def test_bspline_design_device_bit_identical(order):
    from paper_1510_03298_b200 import kronglm as K
    rng = np.random.default_rng(81 + order)
    pts = np.concatenate([[0.0], np.cumsum(rng.uniform(0.2, 1.0, size=300))])
    for nb in (order, order + 3, order + 40):
        host = K.bspline_design(pts, order, nb)
        dev = K.bspline_design_device(pts, order, nb)
        assert host.tobytes() == dev.tobytes()
        assert np.array_equal(O.bspline_design(pts, order, nb), dev)
    grid = np.arange(1.0, 978.0)  # C5's 977-point marginal
    nb = K.default_basis_count(977, 5)
    assert K.bspline_design(grid, order, nb).tobytes() == K.bspline_design_device(grid, order, nb).tobytes()


@pytest.mark.gpu
def test_bspline_design_device_errors():
    from paper_1510_03298_b200 import kronglm as K
    with pytest.raises(ValueError, match="strictly increasing"):
        K.bspline_design_device([0.0, 2.0, 1.0, 3.0], 2, 3)
    with pytest.raises(ValueError, match="at least `order` basis"):
        K.bspline_design_device([0.0, 1.0, 2.0], 4, 3)
    with pytest.raises(ValueError, match="two grid points"):
        K.bspline_design_device([0.0], 1, 1)
