"""The C++ grid engine (csrc/btg_grid_engine.cu) on the GPU, against the oracle:

* NCCL transport at world size 1 (the pool has one GPU per box): the
  multi-process API (ncclCommInitRank) and the single-process one
  (ncclCommInitAll), F / F* / Hessian through the full executor;
* several ranks sharing cuda:0 over the external transport (host callbacks into
  torch.distributed/gloo): 1x2, 2x1, 2x2, 2x3 and a ragged 4x1 grid with an
  empty shard, device shards, the Hessian with a GLOBAL Gamma^-1 (per sensor
  and per sample) and alpha R v — the same schedule the NCCL executor runs;
* the single-process Partition (P2P transport: the reference's tree order on
  the device), its Hessian, serial == parallel, and run-to-run bitwise repeats.
Tolerance: relative L2 <= 1e-12 (FP64, north star)."""

import ctypes
import os
import socket
import tempfile

import numpy as np
import pytest

from oracle import restate as R

pytestmark = pytest.mark.gpu

ND, NM, NT = 7, 40, 32


def _problem():
    blocks, m, d = R.random_problem(33, ND, NM, NT)
    gs = np.linspace(0.5, 2.0, ND)
    gt = np.random.default_rng(4).uniform(0.5, 2.0, size=(ND, NT))
    return blocks, m, d, gs, gt


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _raw_grid_calls(h, m, d, g, L, _lib):
    fwd = np.empty((ND, NT))
    adj = np.empty((NM, NT))
    hes = np.empty((NM, NT))
    _lib.check(L.btg_grid_forward(h, m.ctypes.data, m.size, fwd.ctypes.data, fwd.size, 0))
    _lib.check(L.btg_grid_adjoint(h, d.ctypes.data, d.size, adj.ctypes.data, adj.size, 0))
    _lib.check(L.btg_grid_hessian(h, m.ctypes.data, m.size, hes.ctypes.data, hes.size, g.ctypes.data,
                                  _lib.BTG_GAMMA_PER_SAMPLE, 0.25, _lib.BTG_REG_TEMPORAL_LAPLACIAN, 0))
    return fwd, adj, hes


@pytest.mark.parametrize("mode", ["multiprocess_api", "local_api"])
def test_nccl_transport_world1(mode):
    from paper_2407_13066_b200 import _lib

    L = _lib.load()
    blocks, m, d, _, gt = _problem()
    spec = R.setup_full(blocks)
    h = ctypes.c_void_p()
    if mode == "multiprocess_api":
        uid = ctypes.create_string_buffer(_lib.BTG_NCCL_ID_BYTES)
        _lib.check(L.btg_grid_nccl_id(uid))
        _lib.check(L.btg_grid_create(1, 1, 0, uid.raw, 0, ctypes.byref(h)))
    else:
        devs = (ctypes.c_int * 1)(0)
        _lib.check(L.btg_grid_create_local(1, 1, devs, 1, _lib.BTG_TRANSPORT_NCCL, ctypes.byref(h)))
    try:
        b = np.ascontiguousarray(blocks)
        _lib.check(L.btg_grid_setup(h, b.ctypes.data, ND, NM, NT, 64, 0))
        rows, cols, rank, tr = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_int()
        _lib.check(L.btg_grid_info(h, ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(rank), ctypes.byref(tr)))
        assert (rows.value, cols.value, tr.value) == (1, 1, _lib.BTG_TRANSPORT_NCCL)
        fwd, adj, hes = _raw_grid_calls(h, m, d, gt, L, _lib)
        assert R.rel_l2(fwd, R.apply_forward(spec, m)) <= 1e-12
        assert R.rel_l2(adj, R.apply_adjoint(spec, d)) <= 1e-12
        assert R.rel_l2(hes, R.gauss_newton_apply(spec, m, gt, 0.25, 1)) <= 1e-12
        assert os.environ.get("NCCL_ALGO", "Ring") == "Ring"  # pinned by the library unless the user set it
        # deterministic repeats
        f2, a2, h2 = _raw_grid_calls(h, m, d, gt, L, _lib)
        assert np.array_equal(f2, fwd) and np.array_equal(a2, adj) and np.array_equal(h2, hes)
    finally:
        L.btg_grid_destroy(h)


def _gloo_worker(rank, world, grid, transport, port, outdir):
    import torch
    import torch.distributed as dist

    from paper_2407_13066_b200 import distributed as D

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    blocks, m, d, gs, gt = _problem()
    out = {}
    eng = D.GridEngine.from_blocks(blocks, grid, transport=transport)
    try:
        sh = eng.shard
        dev = torch.device("cuda:0")
        ms = torch.from_numpy(m[sh.source_begin:sh.source_end].copy()).to(dev) if sh.grid_row == 0 else None
        ds = torch.from_numpy(d[sh.sensor_begin:sh.sensor_end].copy()).to(dev) if sh.grid_col == 0 else None
        for rep in range(2):
            f = eng.forward(ms)
            a = eng.adjoint(ds)
            h1 = eng.hessian(ms, alpha=0.3, reg="temporal-laplacian", gamma_inv=torch.from_numpy(gs).to(dev))
            h2 = eng.hessian(ms, alpha=0.0, gamma_inv=torch.from_numpy(gt).to(dev))
            torch.cuda.synchronize()
            for k, v in (("fwd", f), ("adj", a), ("hs", h1), ("ht", h2)):
                if v is not None:
                    out[f"{k}{rep}"] = v.cpu().numpy()
        out["shard"] = np.array([sh.sensor_begin, sh.sensor_end, sh.source_begin, sh.source_end])
        out["bytes"] = np.array([eng.comm_bytes()])
    finally:
        eng.close()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), **out)
    dist.barrier()
    dist.destroy_process_group()


def _assemble(results, key, by_sensor):
    parts = sorted(((int(r["shard"][0 if by_sensor else 2]), r[key]) for r in results if key in r),
                   key=lambda p: p[0])
    return np.concatenate([p[1] for p in parts], axis=0)


@pytest.mark.parametrize("grid", [(1, 2), (2, 1), (2, 2), (2, 3), (4, 1)], ids=lambda g: f"{g[0]}x{g[1]}")
def test_cpp_executor_multi_rank_on_one_gpu(grid):
    """Several ranks on cuda:0, C++ executor, collectives via host callbacks."""
    import torch.multiprocessing as mp

    world = grid[0] * grid[1]
    with tempfile.TemporaryDirectory() as outdir:
        mp.spawn(_gloo_worker, args=(world, grid, "gloo", _free_port(), outdir), nprocs=world, join=True)
        results = [dict(np.load(os.path.join(outdir, f"rank{r}.npz"))) for r in range(world)]
    blocks, m, d, gs, gt = _problem()
    spec = R.setup_full(blocks)
    want = {"fwd": R.apply_forward(spec, m), "adj": R.apply_adjoint(spec, d),
            "hs": R.gauss_newton_apply(spec, m, gs, 0.3, 1), "ht": R.gauss_newton_apply(spec, m, gt, 0.0, 0)}
    for k, w in want.items():
        got = _assemble(results, f"{k}0", by_sensor=(k == "fwd"))
        assert R.rel_l2(got, w) <= 1e-12, k
        assert np.array_equal(got, _assemble(results, f"{k}1", by_sensor=(k == "fwd"))), k  # repeats bitwise
    # the reference's CommLog byte model for one F and one F*
    r, c = grid
    sc, mc = -(-ND // r), -(-NM // c)
    pdims = [min((j + 1) * mc, NM) - min(j * mc, NM) for j in range(c)]
    ddims = [min((i + 1) * sc, ND) - min(i * sc, ND) for i in range(r)]
    one = sum((r - 1) * 8 * NT * x for x in pdims) + sum((c - 1) * 8 * NT * x for x in ddims)
    assert int(results[0]["bytes"][0]) == 2 * 2 * one  # 2 repeats x (F + F*)


def test_nccl_grid_engine_world1():
    """GridEngine (Python shim) over NCCL, torch.distributed world size 1."""
    import torch.multiprocessing as mp

    with tempfile.TemporaryDirectory() as outdir:
        mp.spawn(_gloo_worker, args=(1, (1, 1), "nccl", _free_port(), outdir), nprocs=1, join=True)
        res = dict(np.load(os.path.join(outdir, "rank0.npz")))
    blocks, m, d, gs, gt = _problem()
    spec = R.setup_full(blocks)
    assert R.rel_l2(res["fwd0"], R.apply_forward(spec, m)) <= 1e-12
    assert R.rel_l2(res["adj0"], R.apply_adjoint(spec, d)) <= 1e-12
    assert R.rel_l2(res["hs0"], R.gauss_newton_apply(spec, m, gs, 0.3, 1)) <= 1e-12
    assert R.rel_l2(res["ht0"], R.gauss_newton_apply(spec, m, gt, 0.0, 0)) <= 1e-12


@pytest.mark.parametrize("grid", [(2, 3), (3, 2), (4, 1)])
def test_partition_hessian_p2p(grid):
    """Single-process Partition on the P2P transport: six cells on one device,
    the Hessian schedule with a global Gamma^-1, serial == parallel bitwise."""
    from paper_2407_13066_b200.distributed import Partition

    blocks, m, d, gs, gt = _problem()
    spec = R.setup_full(blocks)
    with Partition(blocks, grid, keep_channel_layout=True) as p:
        h = p.hessian(m, alpha=0.3, reg="temporal-laplacian", gamma_inv=gs)
        assert R.rel_l2(h, R.gauss_newton_apply(spec, m, gs, 0.3, 1)) <= 1e-12
        assert np.array_equal(p.hessian(m, alpha=0.3, reg="temporal-laplacian", gamma_inv=gs, parallel=True), h)
        h2 = p.hessian(m, gamma_inv=gt)
        assert R.rel_l2(h2, R.gauss_newton_apply(spec, m, gt, 0.0, 0)) <= 1e-12
        # the other backends of the local step (Gamma^-1 / alpha R v as separate kernels)
        for backend in ("ewp", "naive"):
            hb = p.hessian(m, alpha=0.3, reg="temporal-laplacian", gamma_inv=gs, backend=backend)
            assert R.rel_l2(hb, R.gauss_newton_apply(spec, m, gs, 0.3, 1)) <= 1e-12, backend


def test_partition_forward_is_reference_tree_of_the_partials():
    """The P2P reduce adds the cells' partials in tree_reduce's order
    (distributed.cpp:36-47): identical bits to tree-summing the shards' own
    single-GPU outputs on the host in that order."""
    import paper_2407_13066_b200 as btg
    from paper_2407_13066_b200.distributed import Partition, partition_bounds

    blocks, m, d, _, _ = _problem()
    grid = (1, 5)
    with Partition(blocks, grid) as p:
        got = p.forward(m)
    parts = []
    for s in partition_bounds(ND, NM, *grid):
        with btg.setup(np.ascontiguousarray(blocks[:, s.sensor_begin:s.sensor_end,
                                                   s.source_begin:s.source_end])) as op:
            parts.append(op.apply_forward(np.ascontiguousarray(m[s.source_begin:s.source_end])))
    assert np.array_equal(got, R.tree_reduce(parts))


@pytest.mark.parametrize("grid,nt", [((2, 3), 64), ((1, 5), 64), ((3, 2), 1024), ((4, 2), 256)])
def test_p2p_reduce_fused_into_c2r_matches_unfused(monkeypatch, grid, nt):
    """P2P transport: a local F / F* followed by a group reduce runs as the
    other members' partials + member 0's C2R loading them (peer access) and
    storing their tree_reduce (C2REpilogue::peers). Same tree, same additions:
    identical bits to the unfused path (BTG_GRID_FUSED=0: receive copies + add
    kernels), for F, F* and the Hessian (row all-reduce) with Gamma^-1 and
    alpha R v."""
    from paper_2407_13066_b200.distributed import Partition

    nd, nm = 7, 29
    blocks, m, d = R.random_problem(41, nd, nm, nt)
    gs = np.linspace(0.5, 2.0, nd)
    out = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("BTG_GRID_FUSED", fused)
        if fused == "1":  # every reduce of these schedules must take the fused path
            monkeypatch.setenv("BTG_GRID_FUSED_REQUIRE", "1")
        with Partition(blocks, grid) as p:
            out[fused] = (p.forward(m), p.adjoint(d), p.hessian(m, alpha=0.3, reg="temporal-laplacian", gamma_inv=gs))
        monkeypatch.delenv("BTG_GRID_FUSED_REQUIRE", raising=False)
    monkeypatch.delenv("BTG_GRID_FUSED", raising=False)
    for a, b in zip(out["1"], out["0"]):
        assert np.array_equal(a, b)
    spec = R.setup_full(blocks)
    f, a, h = out["1"]
    assert R.rel_l2(f, R.apply_forward(spec, m)) <= 1e-12
    assert R.rel_l2(a, R.apply_adjoint(spec, d)) <= 1e-12
    assert R.rel_l2(h, R.gauss_newton_apply(spec, m, gs, 0.3, 1)) <= 1e-12


def test_p2p_fused_reduce_with_empty_cells(monkeypatch):
    """A grid with more rows than the ceiling partition fills (N_d = 5 on 4 rows:
    the last row is empty): column groups fuse with an all-zero member, row
    groups whose member 0 is empty fall back to copies + adds; the results
    equal the unfused path bit for bit and the oracle."""
    from paper_2407_13066_b200.distributed import Partition

    nd, nm, nt = 5, 12, 64
    blocks, m, d = R.random_problem(43, nd, nm, nt)
    out = {}
    for fused in ("1", "0"):
        monkeypatch.setenv("BTG_GRID_FUSED", fused)
        with Partition(blocks, (4, 2)) as p:
            out[fused] = (p.forward(m), p.adjoint(d), p.hessian(m, alpha=0.2))
    monkeypatch.delenv("BTG_GRID_FUSED", raising=False)
    for a, b in zip(out["1"], out["0"]):
        assert np.array_equal(a, b)
    spec = R.setup_full(blocks)
    assert R.rel_l2(out["1"][0], R.apply_forward(spec, m)) <= 1e-12
    assert R.rel_l2(out["1"][1], R.apply_adjoint(spec, d)) <= 1e-12
