"""partition_operator(const SpectralP2O&) on the device (btg_slice_operator):
shards cut from a resident F-hat are bit-identical to the source's blocks, match
the reference's own spectral partition (oracle/_ref, distributed.cpp:198-218),
and their local F / F* reassemble the global matvec."""

import numpy as np
import pytest

from oracle import restate as R
from paper_2407_13066_b200.distributed import partition_bounds

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def btg():
    import paper_2407_13066_b200 as m

    return m


def test_slices_bit_identical_and_match_reference_partition(btg):
    from oracle import refcpu

    nd, nm, nt = 7, 11, 24
    blocks, m, d = R.random_problem(42, nd, nm, nt)
    with btg.setup(blocks) as op:
        full = op.spectrum()
        for rows, cols in [(1, 1), (2, 3), (3, 2), (7, 11), (4, 4)]:
            for sh in partition_bounds(nd, nm, rows, cols):
                if sh.empty:
                    continue
                with op.slice((sh.sensor_begin, sh.sensor_end), (sh.source_begin, sh.source_end)) as s:
                    want = full[:, sh.sensor_begin:sh.sensor_end, sh.source_begin:sh.source_end]
                    assert np.array_equal(s.spectrum(), want)
        if refcpu.available():
            ref = refcpu.RefSpectralOperator(blocks)
            shards = refcpu.spectral_partition_shards(ref, 2, 3)
            for (r, c), (s0, s1, m0, m1, spec) in shards.items():
                with op.slice((s0, s1), (m0, m1)) as s:
                    got = s.freq_blocks
                    assert np.abs(got - spec).max() <= 1e-14 * np.abs(spec).max()


def test_slice_matvecs_reassemble(btg):
    nd, nm, nt = 9, 30, 40
    blocks, m, d = R.random_problem(5, nd, nm, nt)
    spec = R.setup_full(blocks)
    fwd = np.zeros((nd, nt))
    adj = np.zeros((nm, nt))
    with btg.setup(blocks) as op:
        for sh in partition_bounds(nd, nm, 2, 3):
            with op.slice((sh.sensor_begin, sh.sensor_end), (sh.source_begin, sh.source_end)) as s:
                fwd[sh.sensor_begin:sh.sensor_end] += s.apply_forward(m[sh.source_begin:sh.source_end])
                adj[sh.source_begin:sh.source_end] += s.apply_adjoint(d[sh.sensor_begin:sh.sensor_end])
    assert R.rel_l2(fwd, R.apply_forward(spec, m)) <= 1e-12
    assert R.rel_l2(adj, R.apply_adjoint(spec, d)) <= 1e-12


def test_slice_fp32_and_errors(btg):
    blocks, m, d = R.random_problem(8, 4, 10, 16)
    with btg.setup(blocks, precision=32) as op:
        with op.slice((1, 3), (2, 9)) as s:
            assert s.precision == 32
            assert np.array_equal(s.spectrum(), op.spectrum()[:, 1:3, 2:9])
        for bad in [((0, 0), (0, 5)), ((0, 5), (0, 5)), ((0, 2), (3, 11)), ((2, 1), (0, 3))]:
            with pytest.raises(btg.GridError):
                op.slice(*bad)
    # a handle whose rows were never set up cannot be sliced
    with btg.create(4, 10, 16) as op:
        with pytest.raises(btg.Error):
            op.slice((0, 2), (0, 3))
