"""Row- and column-sharded solves on the B200, through the C ABI.

Only one GPU is available per test run, so the sharded schedule is checked
with the engine's in-process loopback group (W host threads, W shard
contexts on one device, collectives as synchronized device copies -- no
kernel waits on another shard) and the NCCL backend at world size 1 (the
real communicator, every collective a no-op exchange).  Checks: all shards
return the same result; the solve meets the north_star bar against the
compiled reference (termination, KKT <= 1e-8, objective within the
admissible gap, first restart period within 1e-10 per iterate)."""
import os
import socket

import numpy as np
import pytest

from paper_2106_04756_b200 import cabi, instances, shard

from _parity import iteration_band

pytestmark = pytest.mark.gpu


def _rel_kkt(info):
    gap = info["gap_abs"] / (1 + abs(info["primal_objective"]) + abs(info["dual_objective"]))
    pr = info["primal_residual_norm"] / (1 + info["norm_q"])
    du = info["dual_residual_norm"] / (1 + info["norm_c"])
    return max(gap, pr, du)


def _same(results):
    a = results[0]
    for b in results[1:]:
        assert b.termination_reason == a.termination_reason
        assert b.iterations == a.iterations and b.restart_iterations == a.restart_iterations
        assert b.final_info == a.final_info
        assert np.array_equal(b.primal_solution, a.primal_solution)
        assert np.array_equal(b.dual_solution, a.dual_solution)


@pytest.mark.parametrize("partition", ["rows", "cols"])
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (5, 0.01)])
def test_loopback_shards_solve_to_1e8(ref, cfg, scale, world, partition):
    lp = instances.generate(cfg, 1, scale)
    p = cabi.params(kkt_pass_limit=300000)
    res = shard.solve_loopback(lp, world, p, partition=partition)
    _same(res)
    a = res[0]
    b = ref.solve_lp(lp, p)
    assert a.termination_reason == b.termination_reason == "Optimal"
    assert _rel_kkt(a.final_info) <= 1e-8
    pa, pb = a.final_info["primal_objective"], b.final_info["primal_objective"]
    assert abs(pa - pb) <= 1e-8 * (2 + 2 * abs(pa) + 2 * abs(pb))
    # tree-order sums: the iteration count moves like that of a re-associated
    # reference (tests/_parity.py iteration_band)
    assert abs(a.iterations - b.iterations) <= iteration_band(cfg, 1, scale) * b.iterations
    assert a.step_condition_violations == 0


@pytest.mark.parametrize("partition", ["rows", "cols"])
@pytest.mark.parametrize("world", [2, 4])
def test_loopback_shards_first_restart_period(ref, world, partition):
    lp = instances.generate(1, 1, 1.0)
    p = cabi.params(record_iterate_trace=True, iteration_limit=100)
    res = shard.solve_loopback(lp, world, p, partition=partition, iterate_capacity=100)
    _same(res)
    b = ref.solve_lp(lp, p, iterate_capacity=100)
    a = res[0]
    assert len(a.iterate_trace) == len(b.iterate_trace) == 100
    worst40 = 0.0
    for (ia, ea, xa, ya), (ib, eb, xb, yb) in zip(a.iterate_trace[:40], b.iterate_trace[:40]):
        assert ia == ib
        for u, v in ((xa, xb), (ya, yb)):
            worst40 = max(worst40, float(np.max(np.abs(u - v) / np.maximum(1.0, np.abs(v)))))
    assert worst40 <= 1e-10
    assert a.restart_iterations == b.restart_iterations
    assert a.kkt_passes == b.kkt_passes


def _loopback_partition(eng, lp, p, world, partition):
    """The partition a `world`-shard loopback session actually runs (the
    engine's own answer, folp_session_partition), checked on every shard
    after one evaluation period."""
    import threading
    g = shard.LoopbackGroup(world)
    out = [None] * world

    def run(r):
        s = eng.session(lp, p, shard=g.spec(r, partition))
        try:
            s.advance(1)
            out[r] = s.partition()
        finally:
            s.close()

    try:
        ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    finally:
        g.close()
    assert out[0] == out[1]
    return out[0]


@pytest.mark.parametrize("cfg,scale,want", [(5, 0.005, "cols"), (3, 0.0005, "rows")])
def test_auto_partition_picks_the_shorter_exchange(eng, cfg, scale, want):
    """AUTO runs columns when m + 2 < n (config 5's shape) and rows otherwise,
    with the same results as the explicit partition."""
    lp = instances.generate(cfg, 1, scale)
    p = cabi.params(iteration_limit=200)
    auto = shard.solve_loopback(lp, 2, p, partition="auto")
    same = shard.solve_loopback(lp, 2, p, partition=want)
    _same(auto + same)
    assert _loopback_partition(eng, lp, p, 2, "auto") == cabi.PARTITIONS[want]
    other = "cols" if want == "rows" else "rows"
    assert _loopback_partition(eng, lp, p, 2, other) == cabi.PARTITIONS[other]


def test_shard_rejects_unsupported_modes():
    lp = instances.generate(1, 1, 0.2)
    with pytest.raises(cabi.FolpError):
        shard.solve_loopback(lp, 2, cabi.params(step_policy="malitsky_pock"))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_nccl_world1_matches_single_gpu(eng):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        lp = instances.generate(1, 1, 1.0)
        p = cabi.params(record_iterate_trace=True, iteration_limit=120)
        a = shard.solve(lp, p, iterate_capacity=120)
    finally:
        dist.destroy_process_group()
    b = eng.solve_lp(lp, p, iterate_capacity=120)
    assert a.iterations == b.iterations == 120
    assert a.restart_iterations == b.restart_iterations
    worst = 0.0
    for (ia, ea, xa, ya), (ib, eb, xb, yb) in zip(a.iterate_trace[:40], b.iterate_trace[:40]):
        for u, v in ((xa, xb), (ya, yb)):
            worst = max(worst, float(np.max(np.abs(u - v) / np.maximum(1.0, np.abs(v)))))
    assert worst <= 1e-12


@pytest.mark.parametrize("partition", ["rows", "cols"])
@pytest.mark.parametrize("world", [2, 3])
def test_peer_exchange_matches_collective(monkeypatch, world, partition):
    """The exchange fused into the partial product's epilogue (each shard
    stores its partial into slot `rank` of every shard's receive area, sums
    in rank order) gives bit-identical solves to the loopback all-reduce
    (which also sums in rank order) -- iterates, restarts and solutions."""
    lp = instances.generate(5, 1, 0.01)
    p = cabi.params(iteration_limit=600, record_iterate_trace=True)
    monkeypatch.setenv("FOLP_SHARD_EPILOGUE", "replicated")  # the same sums as the collective
    monkeypatch.setenv("FOLP_SHARD_EXCHANGE", "peer")
    peer = shard.solve_loopback(lp, world, p, partition=partition, iterate_capacity=50)
    monkeypatch.setenv("FOLP_SHARD_EXCHANGE", "collective")
    coll = shard.solve_loopback(lp, world, p, partition=partition, iterate_capacity=50)
    _same(peer + coll)
    for (ia, ea, xa, ya), (ib, eb, xb, yb) in zip(peer[0].iterate_trace, coll[0].iterate_trace):
        assert ia == ib and ea == eb
        assert np.array_equal(xa, xb) and np.array_equal(ya, yb)


@pytest.mark.parametrize("partition", ["rows", "cols"])
def test_nccl_world1_peer_exchange(eng, monkeypatch, partition):
    """NCCL backend with FOLP_SHARD_EXCHANGE=peer at world size 1: the
    receive area is exported as a CUDA IPC handle, all-gathered through
    NCCL and the fence is the one-element all-reduce -- the multi-GPU code
    path with a single peer (itself)."""
    import torch.distributed as dist
    monkeypatch.setenv("FOLP_SHARD_EXCHANGE", "peer")
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        lp = instances.generate(1, 1, 1.0)
        p = cabi.params(record_iterate_trace=True, iteration_limit=120)
        a = shard.solve(lp, p, partition=partition, iterate_capacity=120)
    finally:
        dist.destroy_process_group()
    b = eng.solve_lp(lp, p, iterate_capacity=120)
    assert a.iterations == b.iterations == 120
    assert a.restart_iterations == b.restart_iterations
    worst = 0.0
    for (ia, ea, xa, ya), (ib, eb, xb, yb) in zip(a.iterate_trace[:40], b.iterate_trace[:40]):
        for u, v in ((xa, xb), (ya, yb)):
            worst = max(worst, float(np.max(np.abs(u - v) / np.maximum(1.0, np.abs(v)))))
    assert worst <= 1e-12


@pytest.mark.parametrize("partition", ["cols", "rows"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_partitioned_epilogue(ref, world, partition, capfd, monkeypatch):
    """The peer exchange with the epilogue on each rank's own range (engine
    ops.cuh OpShardDualOwn for the column partition: dual step on own rows;
    OpShardPrimalOwn for the row partition: primal step on own columns):
    partial products stored to their owner only, the owner sums in rank
    order, the new iterate stored into every rank's vector, the trial sums
    folded in rank order by every rank.  All shards agree bit for bit; the
    first 100 iterates stay within the reference's noise floor with its
    restarts; the solve reaches 1e-8 like the reference (config 5 family:
    W = 8 leaves 12-13 rows per rank)."""
    from _parity import assert_within_floor, reference_floor
    monkeypatch.setenv("FOLP_TIMING", "1")
    lp = instances.generate(5, 1, 0.01)
    p = cabi.params(record_iterate_trace=True, iteration_limit=100)
    res = shard.solve_loopback(lp, world, p, partition=partition, iterate_capacity=100)
    want = "partitioned dual epilogue" if partition == "cols" else "partitioned primal epilogue"
    assert want in capfd.readouterr().err
    _same(res)
    b = ref.solve_lp(lp, p, iterate_capacity=100)
    assert_within_floor(res[0].iterate_trace, b.iterate_trace, reference_floor(lp, p, 100, b), world)
    assert res[0].restart_iterations == b.restart_iterations
    monkeypatch.delenv("FOLP_TIMING")
    p = cabi.params(kkt_pass_limit=300000)
    res = shard.solve_loopback(lp, world, p, partition=partition)
    _same(res)
    a, b = res[0], ref.solve_lp(lp, p)
    assert a.termination_reason == b.termination_reason == "Optimal"
    assert _rel_kkt(a.final_info) <= 1e-8
    pa, pb = a.final_info["primal_objective"], b.final_info["primal_objective"]
    assert abs(pa - pb) <= 1e-8 * (2 + 2 * abs(pa) + 2 * abs(pb))
    assert abs(a.iterations - b.iterations) <= iteration_band(5, 1, 0.01) * b.iterations
