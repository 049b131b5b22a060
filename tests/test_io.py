"""File formats (row f2) against the reference's own reader / writer
(oracle/_ref io::*): byte-identical vector files, time-domain operator files
loaded into HBM, frequency-domain files written in the reference's 2 N_t
layout and read back by the reference, bit-exact round trips (test_io.cpp)."""

import numpy as np
import pytest

from oracle import refcpu
from oracle import restate as R

needs_ref = pytest.mark.skipif(not refcpu.available(), reason="oracle/_ref not built")


@needs_ref
def test_vector_files_byte_identical_with_reference(tmp_path):
    from paper_2407_13066_b200 import io as bio

    v = R.ref_uniform(3, 7 * 11).reshape(7, 11)
    bio.write_vector(tmp_path / "ours.btvc", v)
    refcpu.write_vector(tmp_path / "ref.btvc", v)
    assert (tmp_path / "ours.btvc").read_bytes() == (tmp_path / "ref.btvc").read_bytes()
    np.testing.assert_array_equal(bio.read_vector(tmp_path / "ref.btvc"), v)
    np.testing.assert_array_equal(refcpu.read_vector(tmp_path / "ours.btvc", v.shape), v)
    # TOSI files: (steps, spatial) layout on disk
    bio.write_vector(tmp_path / "tosi.btvc", v.T, ordering="TOSI")
    np.testing.assert_array_equal(bio.read_vector(tmp_path / "tosi.btvc"), v)


def test_bad_files_raise_format_error(tmp_path):
    from paper_2407_13066_b200 import FormatError
    from paper_2407_13066_b200 import io as bio

    (tmp_path / "junk.btop").write_bytes(b"XXXX" + bytes(60))
    with pytest.raises(ValueError):
        bio.peek_operator(tmp_path / "junk.btop")
    (tmp_path / "short.btvc").write_bytes(b"BTVC")
    with pytest.raises(FormatError):
        bio.read_vector(tmp_path / "short.btvc")


@needs_ref
@pytest.mark.gpu
def test_operator_files_round_trip_through_the_reference(tmp_path):
    from paper_2407_13066_b200 import io as bio

    blocks, m, d = R.random_problem(61, 4, 9, 16)
    refcpu.write_compact(tmp_path / "op_time.btop", blocks)
    hdr = bio.peek_operator(tmp_path / "op_time.btop")
    assert hdr["domain"] == "time" and hdr["num_steps"] == 16
    ref = refcpu.RefSpectralOperator(blocks)
    with bio.load_operator(tmp_path / "op_time.btop") as op:
        assert R.rel_l2(op.apply_forward(m), ref.apply_forward(m)) <= 1e-12
        bio.save_operator(op, tmp_path / "op_freq.btop")
        # the reference reads our frequency-domain file and gets its own spectrum back
        spec = refcpu.load_spectral_spectrum(tmp_path / "op_freq.btop", 4, 9, 16)
        assert np.abs(spec - ref.freq_blocks).max() <= 1e-14 * np.abs(ref.freq_blocks).max()
        # bit-exact round trip of our own F-hat through the file
        with bio.load_operator(tmp_path / "op_freq.btop") as op2:
            assert np.array_equal(op2.spectrum(), op.spectrum())
            assert np.array_equal(op2.apply_adjoint(d), op.apply_adjoint(d))
    # a frequency-domain file written by the reference (its 2 N_t layout) loads directly
    refcpu.save_spectral(ref, tmp_path / "ref_freq.btop")
    with bio.load_operator(tmp_path / "ref_freq.btop") as op3:
        assert R.rel_l2(op3.apply_adjoint(d), ref.apply_adjoint(d)) <= 1e-12
    with bio.load_operator(tmp_path / "ref_freq.btop", precision=32) as op4:
        assert R.rel_l2(op4.apply_forward(m), ref.apply_forward(m)) <= 1e-5


@needs_ref
def test_compact_operator_files_byte_identical_with_reference(tmp_path):
    """The module's write_operator / read_operator (bindings.cpp:306-315): our
    time-domain file is byte-identical to the reference's io::write_operator,
    and each side reads the other's file back exactly."""
    import paper_2407_13066_b200 as btg

    blocks, _, _ = R.random_problem(62, 3, 5, 7)
    btg.write_operator(tmp_path / "ours.btop", blocks)
    refcpu.write_compact(tmp_path / "ref.btop", blocks)
    assert (tmp_path / "ours.btop").read_bytes() == (tmp_path / "ref.btop").read_bytes()
    np.testing.assert_array_equal(btg.read_operator(tmp_path / "ref.btop"), blocks)
    # a frequency-domain file is not a compact operator (io.cpp:161-163)
    (tmp_path / "freq.btop").write_bytes(b"BTOP" + (1).to_bytes(4, "little") + (0).to_bytes(4, "little")
                                         + (1).to_bytes(4, "little") + (1).to_bytes(8, "little") * 3
                                         + (1).to_bytes(4, "little") + bytes(20) + bytes(32))
    with pytest.raises(btg.FormatError):
        btg.read_operator(tmp_path / "freq.btop")


def test_planner_cost_helpers_match_reference_formulas():
    """conventional_cost_estimate / apply_arithmetic_intensity (grid_planner.cpp:282-304)."""
    import paper_2407_13066_b200 as btg

    est = btg.conventional_cost_estimate(1e6, 1000, 100, 0.1)
    per = 324.0 * 3e6 * 1000
    assert est["per_solve_flops"] == per
    assert est["effective_rank"] == 100 * 1000 * 0.1
    assert est["conventional_total_flops"] == 2.0 * 1e4 * per
    fft = 100 * per + 2.0 * 1e4 * 8.0 * (1e6 ** (2.0 / 3.0)) * 100 * 1000
    assert est["fft_total_flops"] == pytest.approx(fft, rel=1e-15)
    assert est["ratio"] == pytest.approx(2.0 * 1e4 * per / fft, rel=1e-15)
    with pytest.raises(RuntimeError):
        btg.conventional_cost_estimate(0, 1, 1)
    assert btg.apply_arithmetic_intensity(100, 32768) == pytest.approx(100 * 32768 / (2.0 * (100 * 32768 + 32868)))
