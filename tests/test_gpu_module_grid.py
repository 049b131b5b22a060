"""The reference module's single-process grid entry points,
distributed_forward / distributed_adjoint(blocks, m, grid, backend)
(python/src/bindings.cpp:148-172), on the GPU: against the reference's own
distributed results (tests/golden/distributed_case.npz, test_smoke.py:68-78
grids), with both backends."""

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def btg():
    import paper_2407_13066_b200 as m

    return m


@pytest.mark.parametrize("grid", ["1x4", "2x2", "4x1", "2x3"])
@pytest.mark.parametrize("backend", ["fft", "ewp", "naive"])
def test_module_grid_matches_reference(btg, golden_dir, grid, backend):
    g = np.load(golden_dir / "distributed_case.npz")
    blocks, m, d = R.random_problem(5, 5, 7, 12)
    assert R.rel_l2(btg.distributed_forward(blocks, m, grid, backend), g[f"fwd_{grid}"]) <= 1e-12
    assert R.rel_l2(btg.distributed_adjoint(blocks, d, grid, backend), g[f"adj_{grid}"]) <= 1e-12


def test_module_grid_errors(btg):
    blocks, m, _ = R.random_problem(5, 5, 7, 12)
    with pytest.raises(ValueError):  # GridError: more rows than sensors (distributed.cpp:147-152)
        btg.distributed_forward(blocks, m, "6x1")
    with pytest.raises(RuntimeError):
        btg.distributed_forward(blocks, m, "1x1", backend="blas")
    with pytest.raises(ValueError):
        btg.distributed_forward(blocks, m[:3], "1x2")


def test_naive_backend_matches_reference_naive(btg, golden_dir):
    """naive_apply_forward at configs[0] against the reference's own naive
    result, and the naive adjoint against the FFT adjoint."""
    g = np.load(golden_dir / "config_a_seed1.npz")
    nd, nm, nt = (int(x) for x in g["dims"])
    blocks, m, d = R.random_problem(int(g["seed"]), nd, nm, nt)
    assert R.rel_l2(btg.naive_apply_forward(blocks, m), g["naive_fwd"]) <= 1e-13
    assert R.rel_l2(btg.naive_apply_adjoint(blocks, d), g["adj"]) <= 1e-12
    with pytest.raises(ValueError):
        btg.naive_apply_forward(blocks, m[:, :5])


@pytest.mark.parametrize("parallel", [False, True])
def test_partition_object_serial_parallel_bit_identical(btg, golden_dir, parallel):
    """Partition (distributed.hpp:43-121) over the C ABI: bounds = the reference's,
    serial and parallel (one host thread per cell) bit-identical, both backends."""
    from paper_2407_13066_b200.distributed import Partition

    g = np.load(golden_dir / "distributed_case.npz")
    blocks, m, d = R.random_problem(5, 5, 7, 12)
    with Partition(blocks, "2x3", keep_channel_layout=True) as p:
        assert np.array_equal(np.array(p.bounds()), g["bounds_2x3"])
        f_serial = p.forward(m)
        assert np.array_equal(p.forward(m, parallel=parallel), f_serial)
        assert R.rel_l2(f_serial, g["fwd_2x3"]) <= 1e-12
        assert R.rel_l2(p.adjoint(d, backend="ewp", parallel=parallel), g["adj_2x3"]) <= 1e-12
        assert R.rel_l2(p.adjoint(d, backend="naive", parallel=parallel), g["adj_2x3"]) <= 1e-12


def test_partition_of_a_spectral_operator(btg, golden_dir):
    """partition_operator(SpectralP2O): shards sliced on the device (no re-setup);
    the naive backend is refused like the reference (no time-domain blocks)."""
    from paper_2407_13066_b200.distributed import Partition

    g = np.load(golden_dir / "distributed_case.npz")
    blocks, m, d = R.random_problem(5, 5, 7, 12)
    with btg.setup(blocks) as op, Partition(op, (2, 2)) as p:
        assert R.rel_l2(p.forward(m), g["fwd_2x2"]) <= 1e-12
        assert R.rel_l2(p.adjoint(d), g["adj_2x2"]) <= 1e-12
        with pytest.raises(RuntimeError):
            p.forward(m, backend="naive")
