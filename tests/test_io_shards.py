"""Row f3: shards of a pre-transformed operator without re-running setup.
A rectangle of a frequency-domain file must equal the same rectangle of the
global F-hat bit for bit (test_distributed.cpp:33-45), and a rectangle of a
time-domain file must reproduce it through the local setup."""

import numpy as np
import pytest

from oracle import refcpu
from oracle import restate as R

pytestmark = pytest.mark.gpu


@pytest.mark.skipif(not refcpu.available(), reason="oracle/_ref not built")
def test_rectangles_of_operator_files(tmp_path):
    from paper_2407_13066_b200 import io as bio
    from paper_2407_13066_b200.distributed import partition_bounds

    blocks, m, d = R.random_problem(91, 5, 7, 12)
    refcpu.write_compact(tmp_path / "t.btop", blocks)
    with bio.load_operator(tmp_path / "t.btop") as full:
        bio.save_operator(full, tmp_path / "f.btop")
        spec = full.spectrum()
    for rows, cols in ((2, 3), (1, 4), (3, 2)):
        for s in partition_bounds(5, 7, rows, cols):
            if s.empty:
                continue
            rect = ((s.sensor_begin, s.sensor_end), (s.source_begin, s.source_end))
            want = spec[:, s.sensor_begin:s.sensor_end, s.source_begin:s.source_end]
            with bio.load_operator_rect(tmp_path / "f.btop", *rect) as op:
                assert np.array_equal(op.spectrum(), want)
            with bio.load_operator_rect(tmp_path / "t.btop", *rect) as op:
                assert np.array_equal(op.spectrum(), want)  # per-channel FFT is placement-independent
    with pytest.raises(ValueError):
        bio.load_operator_rect(tmp_path / "f.btop", (0, 6), (0, 7))
