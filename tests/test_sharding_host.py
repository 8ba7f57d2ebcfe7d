"""Host side of the point-sharded path on CPU (world_size 2, gloo): the partition, the exchange
protocol (rank-major all-gather, exact int64 sum) and the report merge.  The device half is in
tests/test_gpu_sharding.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1704_06967_b200 import sharding
from paper_1704_06967_b200.solver import IterationStats, ProblemState, SolveReport
from tests._helpers import random_visibility


def _state(N=23, F=5, keep=0.6, seed=0):
    st = ProblemState(np.zeros((4, 4), np.float32), (1.0, 1.0, 0.0, 0.0), np.zeros((F, 4, 4), np.float32),
                      np.tile([1.0, 1.0, 0.0, 0.0], (F, 1)), np.tile(np.eye(3), (F, 1, 1)), np.zeros((F, 3)),
                      np.arange(2 * N, dtype=np.float64).reshape(N, 2), np.linspace(0.5, 1.5, N),
                      np.array([[0, 0]], np.int32))
    if keep is not None:
        st.obs_ptr, st.obs_frame = random_visibility(st, keep=keep, seed=seed)
    return st


@pytest.mark.parametrize("world", [1, 2, 3, 7])
@pytest.mark.parametrize("keep", [None, 0.4])
def test_partition_covers_every_point_and_observation_once(world, keep):
    st = _state(keep=keep)
    shards = [sharding.shard_problem(st, r, world) for r in range(world)]
    pts = np.concatenate([s.points for s in shards])
    assert np.array_equal(pts, np.arange(st.num_points))
    op = st.obs_ptr if st.obs_ptr is not None else np.arange(st.num_points + 1) * st.num_frames
    of = st.obs_frame if st.obs_frame is not None else np.tile(np.arange(st.num_frames), st.num_points)
    frames = np.concatenate([s.state.obs_frame for s in shards])
    assert np.array_equal(frames, of)
    for s in shards:
        n0, n1 = s.points[0], s.points[-1] + 1
        assert np.array_equal(s.state.obs_ptr, op[n0:n1 + 1] - op[n0])
        assert np.array_equal(s.state.inv_depths, st.inv_depths[n0:n1])
        assert np.array_equal(s.state.anchors_px, st.anchors_px[n0:n1])
        assert s.state.targets is st.targets and s.num_points_total == st.num_points
    # balanced by observations: no shard holds more than its share plus one point's observations
    per = [int(s.state.obs_ptr[-1]) for s in shards]
    kmax = int(np.diff(op).max())
    assert max(per) <= int(op[-1]) / world + kmax


def test_partition_rejects_more_ranks_than_points():
    with pytest.raises(ValueError):
        sharding.shard_bounds(np.arange(4, dtype=np.int64), 5)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x = sharding.TorchExchange()
        assert not x.on_device and (x.rank, x.world) == (rank, world)
        rng = np.random.default_rng(100 + rank)
        part = rng.normal(size=13)
        g = x.gather_host(part)                     # PBA_X_GATHER: rank-major
        # the engine's k_xreduce: fixed rank order, sums and one max slot
        red = g[0].copy()
        for r in range(1, world):
            red[:12] += g[r][:12]
            red[12] = max(red[12], g[r][12])
        big = np.array([2 ** 62, -5, 7 * (rank + 1)], dtype=np.int64)
        s = x.sum_i64_host(big.copy())              # PBA_X_SUM_I64: exact, in place
        q.put((rank, part, g, red, s))
    finally:
        dist.destroy_process_group()


def test_gloo_exchange_protocol_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    out = {}
    for _ in range(world):
        r, part, g, red, s = q.get(timeout=120)
        out[r] = (part, g, red, s)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    parts = np.stack([out[r][0] for r in range(world)])
    for r in range(world):
        assert np.array_equal(out[r][1], parts)                        # every rank sees all, rank-major
        assert np.array_equal(out[r][2].view(np.int64), out[0][2].view(np.int64))  # bitwise identical sums
        assert np.array_equal(out[r][3], out[0][3])                    # the same int64 sum everywhere
    tot = out[0][3]
    assert tot[1] == -10 and tot[2] == 7 + 14
    assert tot[0] == np.int64(-(2 ** 63))  # 2^62 + 2^62 wraps exactly like the device's uint64 accumulator


def test_merge_reports_places_depths_in_caller_order():
    st = _state(N=10, keep=None)
    shards = [sharding.shard_problem(st, r, 3) for r in range(3)]
    reps = []
    for s in shards:
        it = IterationStats(1, 5.0, 0.1, 1.0, 1, 1, num_active=100,
                            inv_depths=-s.points.astype(np.float64))
        reps.append(SolveReport(iters=[it], iterations=1, final_energy=5.0, final_R=np.zeros((5, 3, 3)),
                                final_t=np.zeros((5, 3)), final_inv_depths=s.points.astype(np.float64) * 2,
                                masked_residuals=4, total_wall_ms=float(s.rank)))
    m = sharding.merge_reports(shards, reps)
    assert np.array_equal(m.final_inv_depths, np.arange(10) * 2.0)
    assert np.array_equal(m.iters[0].inv_depths, -np.arange(10.0))
    # energies and counts are the exchanged global sums on every rank: taken from rank 0, not re-summed
    assert m.iters[0].num_active == 100 and m.masked_residuals == 4 and m.total_wall_ms == 2.0


def test_merge_warnings_frames_once_points_in_caller_order():
    """frame warnings come from one shard (every shard raises them), zero-depth points are
    mapped from each shard's local indices to caller indices (solver.cpp:265-271, 359-364)."""
    from paper_1704_06967_b200.solver import WarningList
    st = _state(N=10, keep=None)
    shards = [sharding.shard_problem(st, r, 3) for r in range(3)]
    head = ["frame 2: zero initial translation, inverse depth unobservable from this frame"]
    local = [np.array([0], np.int32), np.zeros(0, np.int32), np.array([0, len(shards[2].points) - 1], np.int32)]
    parts = [WarningList(head, p) for p in local]
    m = sharding.merge_warnings(shards, parts)
    want = [int(shards[0].points[0]), int(shards[2].points[0]), int(shards[2].points[-1])]
    assert list(m) == head + [f"point {i}: zero depth Hessian entry (unobservable depth)" for i in want]
    # plain string lists (a checker library's report) merge the same way
    assert list(sharding.merge_warnings(shards, [list(p) for p in parts])) == list(m)
