"""Multi-process tests of the 2-D grid engine on CPU: torch.distributed with
the gloo backend, one process per grid cell, world sizes 2, 4 and 6.

What is under test is the PRODUCT's choreography: every rank fetches its step
list from libbtg (btg_grid_schedule — the same schedule the C++ executor runs
with NCCL) and executes it here with gloo collectives and a host stand-in for
the shard-local compute built on the oracle (test infrastructure). Results are
checked against the reference's own distributed results
(tests/golden/distributed_case.npz, produced by oracle/_ref's
distributed_forward / distributed_adjoint) and the reference's CommLog byte
model (test_distributed.cpp:139-204). The C++ executor itself (device shards,
the external / NCCL transports) is covered by the GPU tests below and in
tests/test_gpu_grid.py."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restate as R
from paper_2407_13066_b200 import _lib
from paper_2407_13066_b200 import distributed as D

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "distributed_case.npz")


class OracleLocalOp:
    """Host stand-in for a shard's operator: F with an optional Gamma^-1 row
    scaling, F* with an optional + alpha R v (the C2R epilogues)."""

    def __init__(self, blocks):
        self.spec = R.setup_full(blocks)

    def forward(self, x, gamma=None):
        y = R.apply_forward(self.spec, x)
        if gamma is not None:
            y = y * (gamma[:, None] if gamma.ndim == 1 else gamma)
        return y

    def adjoint(self, y, reg_v=None, alpha=0.0, reg_kind=0):
        x = R.apply_adjoint(self.spec, y)
        if reg_v is not None and alpha != 0.0:
            x = x + alpha * R.reg_apply(reg_v, reg_kind)
        return x


def run_schedule(kind, grid, rank, shard, local, x_slice, nt, groups, gamma=None, alpha=0.0, reg_kind=0,
                 nd=None, nm=None):
    """Execute libbtg's step list for this rank with gloo + the host stand-in."""
    steps = D.schedule(nd, nm, nt, grid, rank, kind, with_gamma=gamma is not None, with_reg=alpha != 0.0)
    rows, cols = grid
    i, j = divmod(rank, cols)
    row_groups, col_groups = groups
    bufs = {}
    result = None
    for s in steps:
        op = s["op"]
        if op == _lib.BTG_STEP_INPUT:
            if s["active"]:
                assert x_slice is not None and x_slice.size == s["count"]
                bufs[s["dst"]] = np.array(x_slice, dtype=np.float64)
            else:
                bufs[s["dst"]] = np.zeros(s["count"] // nt * nt).reshape(-1, nt)
        elif op in (_lib.BTG_STEP_BROADCAST, _lib.BTG_STEP_REDUCE, _lib.BTG_STEP_ALLREDUCE):
            row = s["group"] == _lib.BTG_GROUP_ROW
            grp = row_groups[i] if row else col_groups[j]
            root = i * cols + s["root"] if row else s["root"] * cols + j
            t = torch.from_numpy(np.ascontiguousarray(bufs[s["src"]]).reshape(-1))
            if t.numel():
                if op == _lib.BTG_STEP_BROADCAST:
                    dist.broadcast(t, src=root, group=grp)
                elif op == _lib.BTG_STEP_REDUCE:
                    dist.reduce(t, dst=root, group=grp)
                else:
                    dist.all_reduce(t, group=grp)
            bufs[s["src"]] = t.numpy().reshape(-1, nt)
        elif op == _lib.BTG_STEP_FORWARD:
            g = gamma[shard.sensor_begin:shard.sensor_end] if (s["gamma"] and gamma is not None) else None
            bufs[s["dst"]] = (local.forward(bufs[s["src"]], g) if local is not None
                              else np.zeros((shard.local_sensors, nt)))
            assert bufs[s["dst"]].size == s["count"]
        elif op == _lib.BTG_STEP_ADJOINT:
            rv = bufs[0] if s["reg"] else None
            bufs[s["dst"]] = (local.adjoint(bufs[s["src"]], rv, alpha, reg_kind) if local is not None
                              else np.zeros((shard.local_sources, nt)))
            assert bufs[s["dst"]].size == s["count"]
        elif op == _lib.BTG_STEP_OUTPUT:
            if s["active"]:
                result = bufs[s["src"]]
    return result


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, grids, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blocks, m, d = R.random_problem(5, 5, 7, 12)
    gamma = np.linspace(0.5, 2.0, 5)
    results = {}
    for grid in grids:
        rows, cols = grid
        row_groups = [dist.new_group([i * cols + j for j in range(cols)]) for i in range(rows)]
        col_groups = [dist.new_group([i * cols + j for i in range(rows)]) for j in range(cols)]
        shard = D.partition_bounds(5, 7, *grid)[rank]
        local = None
        if not shard.empty:
            local = OracleLocalOp(blocks[:, shard.sensor_begin:shard.sensor_end, shard.source_begin:shard.source_end])
        i, j = shard.grid_row, shard.grid_col
        m_slice = m[shard.source_begin:shard.source_end].copy() if i == 0 else None
        d_slice = d[shard.sensor_begin:shard.sensor_end].copy() if j == 0 else None
        key = f"{grid[0]}x{grid[1]}"
        common = dict(grid=grid, rank=rank, shard=shard, local=local, nt=12, groups=(row_groups, col_groups),
                      nd=5, nm=7)
        fwd = run_schedule("forward", x_slice=m_slice, **common)
        adj = run_schedule("adjoint", x_slice=d_slice, **common)
        hes = run_schedule("hessian", x_slice=m_slice, gamma=gamma, alpha=0.3, reg_kind=1, **common)
        if fwd is not None:
            results[f"fwd_{key}"] = fwd
        if adj is not None:
            results[f"adj_{key}"] = adj
            results[f"hes_{key}"] = hes
        log = D.comm_events(5, 7, 12, grid, "forward") + D.comm_events(5, 7, 12, grid, "adjoint")
        results[f"bytes_{key}"] = np.array([sum(e.total_bytes for e in log)])
        results[f"shard_{key}"] = np.array([shard.sensor_begin, shard.sensor_end, shard.source_begin,
                                            shard.source_end])
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **results)
    dist.barrier()
    dist.destroy_process_group()


def _run(world, grids):
    with tempfile.TemporaryDirectory() as outdir:
        mp.spawn(_worker, args=(world, grids, _free_port(), outdir), nprocs=world, join=True)
        return [dict(np.load(os.path.join(outdir, f"rank{r}.npz"))) for r in range(world)]


def _assemble(results, key, kind):
    parts = []
    for r in results:
        if f"{kind}_{key}" in r:
            s = r[f"shard_{key}"]
            begin = s[0] if kind == "fwd" else s[2]
            parts.append((begin, r[f"{kind}_{key}"]))
    parts.sort(key=lambda p: p[0])
    return np.concatenate([p[1] for p in parts], axis=0)


def _check(results, grids):
    g = np.load(GOLDEN)
    blocks, m, d = R.random_problem(5, 5, 7, 12)
    spec = R.setup_full(blocks)
    gamma = np.linspace(0.5, 2.0, 5)
    want_h = R.gauss_newton_apply(spec, m, gamma, 0.3, 1)
    for grid in grids:
        key = f"{grid[0]}x{grid[1]}"
        fwd = _assemble(results, key, "fwd")
        adj = _assemble(results, key, "adj")
        hes = _assemble(results, key, "hes")
        assert R.rel_l2(fwd, R.apply_forward(spec, m)) <= 1e-12
        assert R.rel_l2(adj, R.apply_adjoint(spec, d)) <= 1e-12
        assert R.rel_l2(hes, want_h) <= 1e-12
        if f"fwd_{key}" in g:  # the reference's own distributed engine on the same grid
            assert R.rel_max_diff(fwd, g[f"fwd_{key}"]) < 1e-12
            assert R.rel_max_diff(adj, g[f"adj_{key}"]) < 1e-12
            want_bounds = [tuple(b) for b in g[f"bounds_{key}"]]
            got_bounds = [tuple(int(x) for x in r[f"shard_{key}"]) for r in results]
            assert got_bounds == want_bounds
        # CommLog model: broadcast + reduce payloads per F and F* (distributed.cpp:23-34)
        r, c = grid
        nt = 12
        expect = 0
        for phase_participants, dims in (((r,), _param_dims(7, c)), ((c,), _data_dims(5, r)),
                                         ((c,), _data_dims(5, r)), ((r,), _param_dims(7, c))):
            expect += sum((phase_participants[0] - 1) * 8 * nt * dd for dd in dims)
        assert int(results[0][f"bytes_{key}"][0]) == expect


def _param_dims(nm, cols):
    return [s.local_sources for s in D.partition_bounds(nm, nm, 1, cols)]


def _data_dims(nd, rows):
    return [s.local_sensors for s in D.partition_bounds(nd, nd, rows, 1)]


def test_partition_bounds_match_reference():
    g = np.load(GOLDEN)
    for key in ("1x4", "2x2", "4x1", "2x3"):
        r, c = map(int, key.split("x"))
        got = [(s.sensor_begin, s.sensor_end, s.source_begin, s.source_end) for s in D.partition_bounds(5, 7, r, c)]
        assert got == [tuple(b) for b in g[f"bounds_{key}"]]
    with pytest.raises(ValueError):
        D.partition_bounds(2, 3, 3, 1)
    with pytest.raises(ValueError):
        D.partition_bounds(2, 3, 1, 4)
    # ragged: trailing shard smaller; empty trailing shards allowed
    s = D.partition_bounds(5, 4, 2, 1)
    assert (s[0].local_sensors, s[1].local_sensors) == (3, 2)
    s = D.partition_bounds(5, 7, 4, 1)
    assert [x.local_sensors for x in s] == [2, 2, 1, 0] and s[3].empty


def test_grid_world2():
    grids = [(1, 2), (2, 1)]
    _check(_run(2, grids), grids)


def test_grid_world4():
    grids = [(2, 2), (1, 4), (4, 1)]
    _check(_run(4, grids), grids)


def test_grid_world6():
    grids = [(2, 3), (3, 2)]
    _check(_run(6, grids), grids)


def test_schedule_shapes():
    """Every rank of every factorisation of 8 (and ragged / empty-shard grids)
    gets the same step ops; collectives over one-member groups are omitted."""
    for nd, nm, grids in ((600, 8192, [(1, 8), (2, 4), (4, 2), (8, 1)]), (5, 7, [(4, 1), (2, 3), (3, 2)])):
        for grid in grids:
            for kind in ("forward", "adjoint", "hessian"):
                ops = None
                for rank in range(grid[0] * grid[1]):
                    st = D.schedule(nd, nm, 10, grid, rank, kind, with_gamma=True, with_reg=True)
                    seq = [s["op"] for s in st]
                    ops = ops or seq
                    assert seq == ops
                    assert st[0]["op"] == _lib.BTG_STEP_INPUT and st[-1]["op"] == _lib.BTG_STEP_OUTPUT
                coll = [s for s in D.schedule(nd, nm, 10, grid, 0, kind) if s["op"] in (1, 4, 5)]
                for s in coll:
                    members = grid[1] if s["group"] == _lib.BTG_GROUP_ROW else grid[0]
                    assert members > 1
    with pytest.raises(ValueError):
        D.schedule(5, 7, 12, (2, 2), 4, "forward")
