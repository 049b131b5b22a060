"""Grid planner (native, btg_select_grid & co.) against the reference's own
grid_planner.cpp compiled in oracle/_ref, plus the reference's planner test
expectations (test_grid_planner.cpp). CPU only: pure host arithmetic."""

import math

import numpy as np
import pytest

import paper_2407_13066_b200 as btg
from oracle import refcpu


needs_ref = pytest.mark.skipif(not refcpu.available(), reason="oracle/_ref not built")


@needs_ref
def test_select_grid_matches_reference_sweep():
    rng = np.random.default_rng(3)
    ls = np.concatenate([np.linspace(-4, 4, 81), rng.uniform(-6, 6, 60), [0.0, -2.4, math.log10(600 / 8192)]])
    for p in [1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 97, 128]:
        for k in [1, 2, 4, 8]:
            for l in ls:
                assert btg.select_grid(p, float(l), k) == refcpu.select_grid(p, float(l), k), (p, l, k)


@needs_ref
def test_costs_match_reference():
    for p in [2, 8, 48]:
        for l in [-3.0, -0.5, 0.0, 1.7]:
            for r in [1.0, 1.5, 2.0, p / 2, float(p)]:
                assert btg.modified_cost(r, p, l) == pytest.approx(refcpu.modified_cost(r, p, l), rel=1e-15)
    for (r, c) in [(1, 8), (2, 4), (4, 2), (8, 1), (3, 5)]:
        for dims in [(65536, 256, 4096), (8192, 600, 1000), (10, 10, 7)]:
            want = refcpu.comm_cost(r, c, *dims, latency=2e-6, bandwidth=9e11)
            got = btg.comm_cost((r, c), *dims, latency=2e-6, bandwidth=9e11)
            assert got == pytest.approx(want, rel=1e-15)


@needs_ref
def test_weak_scaling_matches_reference():
    for ratio in [1e-3, 600 / 8192, 0.5, 1.0, 2.0, 37.0]:
        for p in [1, 2, 8]:
            assert btg.weak_scaling_shape(ratio, p) == refcpu.weak_scaling_shape(ratio, p)


def test_planner_picks_for_survey_configs():
    # C (600 x 8192 per GPU) -> 1x8 by weak_scaling_shape; E (256 x 65536) -> 1x8
    assert btg.weak_scaling_shape(600 / 8192, 8) == (False, (1, 8))
    assert btg.plan_grid(256, 65536, 8) == (1, 8)
    assert btg.plan_grid(256, 65536, 8, gpus_per_node=8) == (1, 8)
    assert btg.select_grid(1, 0.3) == (1, 1)
    assert btg.weak_scaling_shape(1.0, 4) == (True, (1, 4))


def test_planner_errors():
    with pytest.raises(btg.Error):
        btg.select_grid(0, 0.0)
    with pytest.raises(btg.Error):
        btg.select_grid(4, 0.0, 0)
    with pytest.raises(btg.Error):
        btg.modified_cost(0.5, 4, 0.0)
    with pytest.raises(btg.Error):
        btg.weak_scaling_shape(0.0, 4)
    with pytest.raises(btg.Error):
        btg.comm_cost((2, 2), 4, 4, 4, bandwidth=0.0)
    assert btg.parse_grid("2x4") == (2, 4) and btg.parse_grid("8X1") == (8, 1)
    for bad in ["2", "x4", "2x", "0x3", "axb"]:
        with pytest.raises(btg.Error):
            btg.parse_grid(bad)


def test_reference_planner_cases():
    """test_grid_planner.cpp:32-118 replayed on the native planner."""
    assert btg.comm_cost((1, 1), 100, 10, 50) == 0.0
    assert btg.modified_cost(80.0, 80, -2.0) == pytest.approx(math.log(80.0), rel=1e-14)
    with pytest.raises(btg.Error):
        btg.modified_cost(5.0, 4, 0.0)
    costs = {r: btg.modified_cost(float(r), 80, -2.0) for r in range(1, 81) if 80 % r == 0}
    best_rows = min(costs, key=costs.get)
    assert best_rows == 2 and costs[2] < btg.modified_cost(1.0, 80, -2.0)
    assert btg.select_grid(48, -3.0, 1) == (1, 48)
    assert btg.select_grid(48, -3.0, 3) == (1, 48)
    assert btg.select_grid(80, -2.0, 4) == (4, 20)
    assert btg.select_grid(80, -3.0, 4) == (1, 80)
    assert btg.select_grid(80, -4.0, 4) == (1, 80)
    # one GPU per node: the integer minimiser (brute force, test_grid_planner.cpp:102-111)
    for p in range(1, 65):
        for l in range(-4, 5):
            r, c = btg.select_grid(p, float(l), 1)
            assert r * c == p
            brute = min(btg.modified_cost(float(q), p, float(l)) for q in range(1, p + 1) if p % q == 0)
            assert btg.modified_cost(float(r), p, float(l)) <= brute * (1 + 1e-12)
    assert btg.weak_scaling_shape(2.0, 6) == (False, (6, 1))
    assert btg.weak_scaling_shape(0.1, 6) == (False, (1, 6))


def test_b200_planner_costs_the_schedule():
    """btg_plan_grid: every factorisation costed, the pick is the cheapest;
    configs[4] (N_d << N_m) goes 1 x 8; a square operator goes 2-D (the replicated
    vector transforms shrink with both cuts); inter-node groups cost more."""
    from paper_2407_13066_b200.planner import default_hw_model, plan_grid_b200

    best, table = plan_grid_b200(256, 65536, 4096, 8, "hessian")
    assert [(t["rows"], t["cols"]) for t in table] == [(1, 8), (2, 4), (4, 2), (8, 1)]
    assert best == (1, 8)
    assert min(table, key=lambda t: t["seconds"])["rows"] == best[0]
    for t in table:
        assert t["seconds"] == pytest.approx(t["local_seconds"] + t["comm_seconds"])
    best_sq, tsq = plan_grid_b200(65536, 65536, 1024, 8, "hessian")
    assert best_sq[0] > 1 and best_sq[1] > 1
    # configs[2] weak-scaling shape at 8 GPUs (global 600 x 65536): 1 x 8, as the reference's rule
    assert plan_grid_b200(600, 8 * 8192, 1000, 8, "forward")[0] == (1, 8)
    # a slow inter-node link makes grids whose groups leave the NVSwitch domain dearer
    _, t16 = plan_grid_b200(4096, 4096, 1024, 16, "hessian", hw={"gpus_per_node": 8})
    _, t16b = plan_grid_b200(4096, 4096, 1024, 16, "hessian", hw={"gpus_per_node": 16})
    assert sum(t["comm_seconds"] for t in t16) > sum(t["comm_seconds"] for t in t16b)
    assert default_hw_model()["gpus_per_node"] == 8
    # grids wider than the operator are not offered; none fits -> GridError
    _, small = plan_grid_b200(2, 3, 8, 4, "forward")
    assert [(t["rows"], t["cols"]) for t in small] == [(2, 2)]
    with pytest.raises(btg.GridError):
        plan_grid_b200(1, 1, 8, 4, "forward")
