"""Point-sharded solves on the device against the oracle's single-process solve of the
whole problem.  Several shards of one process share the GPU (one host thread and handle each);
they meet only at the host-staged exchange, their kernels never wait on one another.  The NCCL
path (zero-copy on the handle's stream) is exercised at world size 1."""
from __future__ import annotations

import os
import socket
from pathlib import Path

import numpy as np
import pytest

from paper_1704_06967_b200 import scenes, sharding, solver
from paper_1704_06967_b200.solver import Handle, OutOfBounds

from ._helpers import random_visibility
from .test_gpu_parity import _compare_runs
from ._oracle import ORACLE

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1():
    return scenes.make_scene(scenes.baseline_config("C1"), device="cpu")


def _runs_equal_bitwise(a, b):
    assert a.iterations == b.iterations and a.final_energy == b.final_energy
    assert [s.energy for s in a.iters] == [s.energy for s in b.iters]
    assert np.array_equal(a.final_inv_depths, b.final_inv_depths)
    assert np.array_equal(a.final_R, b.final_R) and np.array_equal(a.final_t, b.final_t)


@pytest.mark.parametrize("solver_kind", ["ic", "fc"])
def test_one_shard_through_the_exchange_is_bitwise_the_single_process_solve(c1, solver_kind):
    st = c1.state
    cfg = c1.cfg.solver_config(max_iters=4)
    one = sharding.solve_threads(st, cfg, 1, solver_kind)
    h = Handle(st, "gpu")
    ref = h.ic_run(cfg) if solver_kind == "ic" else h.fc_run(cfg)
    _runs_equal_bitwise(one, ref)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("solver_kind", ["ic", "fc"])
def test_sharded_run_matches_oracle_c1(c1, world, solver_kind):
    st = c1.state
    cfg = c1.cfg.solver_config()  # 10 LM iterations
    rg = sharding.solve_threads(st, cfg, world, solver_kind)
    o = Handle(st, ORACLE)
    ro = o.ic_run(cfg) if solver_kind == "ic" else o.fc_run(cfg)
    if solver_kind == "ic":
        assert rg.hessian_builds == 1
    _compare_runs(rg, ro, st.num_frames, st.num_points)


def test_sharded_run_partial_visibility_matches_oracle(c1):
    st = c1.state.copy()
    st.obs_ptr, st.obs_frame = random_visibility(st, 0.6, seed=9)
    cfg = c1.cfg.solver_config(max_iters=5, record_snapshots=True)
    rg = sharding.solve_threads(st, cfg, 2, "ic")
    ro = Handle(st, ORACLE).ic_run(cfg)
    _compare_runs(rg, ro, st.num_frames, st.num_points)
    for a, b in zip(rg.iters, ro.iters):  # merged per-iteration depth snapshots in caller order
        assert np.linalg.norm(a.inv_depths - b.inv_depths) <= 1e-4 * np.linalg.norm(b.inv_depths)


def test_sharded_errors_are_raised_on_every_shard(c1):
    st = c1.state.copy()
    st.anchors_px = st.anchors_px.copy()
    st.anchors_px[-1] = (0.0, 0.0)  # template outside the margin, in the last shard only
    with pytest.raises(OutOfBounds):
        sharding.solve_threads(st, c1.cfg.solver_config(max_iters=2), 2, "ic")


def test_nccl_exchange_world1_is_bitwise_the_single_process_solve(c1):
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        st = c1.state
        cfg = c1.cfg.solver_config(max_iters=4)
        for kind in ("ic", "fc"):
            rg = sharding.solve_distributed(st, cfg, kind)
            h = Handle(st, "gpu")
            ref = h.ic_run(cfg) if kind == "ic" else h.fc_run(cfg)
            _runs_equal_bitwise(rg, ref)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_warnings_match_the_single_process_solve(c1, world):
    """Frame warnings once, zero-depth warnings in caller point order (IcSolver::warnings(),
    solver.cpp:265-271, 359-364): a frame with zero initial translation and points without any
    observation spread over every shard."""
    st = c1.state.copy()
    op, of = random_visibility(st, 0.7, seed=4)
    keep = np.ones(st.num_points, bool)
    keep[::97] = False  # unobserved points: D_n = 0
    cnt = np.diff(op) * keep
    st.obs_ptr = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
    st.obs_frame = np.concatenate([of[op[n]:op[n + 1]] for n in range(st.num_points) if keep[n]]).astype(np.int32)
    st.t = st.t.copy()
    st.t[3] = 0.0
    cfg = c1.cfg.solver_config(max_iters=2)
    one = Handle(st, "gpu").ic_run(cfg)
    ro = Handle(st, ORACLE).ic_run(cfg)
    assert list(one.warnings) == list(ro.warnings)
    assert len(one.warnings) == 1 + int((~keep).sum())
    rg = sharding.solve_threads(st, cfg, world, "ic")
    assert list(rg.warnings) == list(one.warnings)


def test_two_process_gloo_sharded_solve_matches_oracle(tmp_path):
    """a full point-sharded IC and FC solve by two PROCESSES (torch.distributed,
    gloo, world size 2) on one GPU, merged and compared with the oracle's single-process solve."""
    import json
    import subprocess
    import sys
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    worker = Path(__file__).resolve().parent / "mp_sharded_worker.py"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(worker), str(tmp_path)]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    res = json.loads((tmp_path / "rank0.json").read_text())
    for kind in ("ic", "fc"):
        r = res[kind]
        assert r["world"] == 2 and r["control_flow_and_energies"], r
        assert r["params"] is True, r
        assert r["warnings_equal"], r


def test_library_nccl_exchange_world1_is_bitwise_the_single_process_solve(c1):
    """pba_gpu_set_exchange_nccl: the library's own NCCL communicator (collectives on the handle's
    stream, no callback per candidate) at world size 1 reproduces the single-process solve bitwise."""
    import torch
    import torch.distributed as dist
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        st = c1.state
        cfg = c1.cfg.solver_config(max_iters=4)
        for kind in ("ic", "fc"):
            rg = sharding.solve_distributed(st, cfg, kind, exchange="nccl-lib")
            h = Handle(st, "gpu")
            ref = h.ic_run(cfg) if kind == "ic" else h.fc_run(cfg)
            _runs_equal_bitwise(rg, ref)
    finally:
        dist.destroy_process_group()
