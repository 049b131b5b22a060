"""Multi-process tests of the 2-D grid engine (paper_2407_13066_b200.distributed)
on CPU: torch.distributed with the gloo backend, one process per grid cell,
world sizes 2, 4 and 6. The shard-local compute is a host stand-in built on the
oracle (test infrastructure); what is under test is the product's partition,
collective pattern, slice ownership and Hessian composition, checked against
the reference's own distributed results (tests/golden/distributed_case.npz,
produced by oracle/_ref's distributed_forward / distributed_adjoint) and the
reference's CommLog byte model (test_distributed.cpp:139-204)."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import restate as R
from paper_2407_13066_b200 import distributed as D

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "distributed_case.npz")


class OracleLocalOp:
    """Host stand-in for a shard's SpectralOperator (same method signatures)."""

    def __init__(self, blocks):
        self.spec = R.setup_full(blocks)

    def apply_forward(self, x, gamma_inv=None):
        y = R.apply_forward(self.spec, x.numpy())
        if gamma_inv is not None:
            g = gamma_inv.numpy()
            y = y * (g[:, None] if g.ndim == 1 else g)
        return torch.from_numpy(y)

    def apply_adjoint(self, y, reg_v=None, alpha=0.0, reg="identity"):
        x = R.apply_adjoint(self.spec, y.numpy())
        if reg_v is not None and alpha != 0.0:
            x = x + alpha * R.reg_apply(reg_v.numpy(), 0 if reg == "identity" else 1)
        return torch.from_numpy(x)


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
        shard = D.partition_bounds(5, 7, *grid)[rank]
        local = None
        if not shard.empty:
            local = OracleLocalOp(blocks[:, shard.sensor_begin:shard.sensor_end, shard.source_begin:shard.source_end])
        eng = D.GridEngine(5, 7, 12, grid, local)
        i, j = shard.grid_row, shard.grid_col
        m_slice = torch.from_numpy(m[shard.source_begin:shard.source_end].copy()) if i == 0 else None
        d_slice = torch.from_numpy(d[shard.sensor_begin:shard.sensor_end].copy()) if j == 0 else None
        key = f"{grid[0]}x{grid[1]}"
        fwd = eng.forward(m_slice)
        adj = eng.adjoint(d_slice)
        hes = eng.hessian(m_slice, alpha=0.3, reg="temporal-laplacian", gamma_inv=torch.from_numpy(gamma))
        if fwd is not None:
            results[f"fwd_{key}"] = fwd.numpy()
        if adj is not None:
            results[f"adj_{key}"] = adj.numpy()
            results[f"hes_{key}"] = hes.numpy()
        results[f"bytes_{key}"] = np.array([eng.comm_bytes()])
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


class GpuShardOp:
    """The product's shard operator (libbtg on cuda:0) behind host tensors, so
    the engine's gloo collectives run on CPU while the shard compute is CUDA."""

    def __init__(self, blocks):
        import paper_2407_13066_b200 as btg

        self.op = btg.setup(blocks, device=0)

    def apply_forward(self, x, gamma_inv=None):
        g = None if gamma_inv is None else gamma_inv.cuda()
        return self.op.apply_forward(x.cuda(), gamma_inv=g).cpu()

    def apply_adjoint(self, y, reg_v=None, alpha=0.0, reg="identity"):
        rv = None if reg_v is None else reg_v.cuda()
        return self.op.apply_adjoint(y.cuda(), reg_v=rv, alpha=alpha, reg=reg).cpu()

    def close(self):
        self.op.close()


def _gpu_worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blocks, m, d = R.random_problem(21, 6, 40, 32)
    out = {}
    for grid in ((1, 2), (2, 1)):
        shard = D.partition_bounds(6, 40, *grid)[rank]
        local = GpuShardOp(blocks[:, shard.sensor_begin:shard.sensor_end, shard.source_begin:shard.source_end])
        eng = D.GridEngine(6, 40, 32, grid, local)
        i, j = shard.grid_row, shard.grid_col
        ms = torch.from_numpy(m[shard.source_begin:shard.source_end].copy()) if i == 0 else None
        ds = torch.from_numpy(d[shard.sensor_begin:shard.sensor_end].copy()) if j == 0 else None
        key = f"{grid[0]}x{grid[1]}"
        f = eng.forward(ms)
        a = eng.adjoint(ds)
        h = eng.hessian(ms, alpha=0.1, reg="identity", gamma_inv=torch.linspace(0.5, 2.0, 6, dtype=torch.float64))
        if f is not None:
            out[f"fwd_{key}"] = f.numpy()
        if a is not None:
            out[f"adj_{key}"] = a.numpy()
            out[f"hes_{key}"] = h.numpy()
        out[f"shard_{key}"] = np.array([shard.sensor_begin, shard.sensor_end, shard.source_begin, shard.source_end])
        eng.close()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_grid_world2_with_cuda_shards():
    with tempfile.TemporaryDirectory() as outdir:
        mp.spawn(_gpu_worker, args=(2, _free_port(), outdir), nprocs=2, join=True)
        results = [dict(np.load(os.path.join(outdir, f"rank{r}.npz"))) for r in range(2)]
    blocks, m, d = R.random_problem(21, 6, 40, 32)
    spec = R.setup_full(blocks)
    want_h = R.gauss_newton_apply(spec, m, np.linspace(0.5, 2.0, 6), 0.1, 0)
    for key in ("1x2", "2x1"):
        assert R.rel_l2(_assemble(results, key, "fwd"), R.apply_forward(spec, m)) <= 1e-12
        assert R.rel_l2(_assemble(results, key, "adj"), R.apply_adjoint(spec, d)) <= 1e-12
        assert R.rel_l2(_assemble(results, key, "hes"), want_h) <= 1e-12
