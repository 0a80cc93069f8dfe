"""Host logic of the multi-GPU shards, no GPU needed:
the row partition (folp_gpu_shard_rows), the per-shard CSC extraction
(folp_gpu_shard_local_csc), the column partition's CSR extraction
(folp_gpu_shard_local_csr), and -- with two gloo processes on 127.0.0.1 --
the exchange algebra of the sharded trials: the all-reduced partial products
K'_p y_p equal K'y, and the shards' K_p x slices reassemble K x (the
reassembly the engine does by broadcasting each shard's rows); for the
column partition the all-reduced K_p x_p equal K x and the shards' x blocks
reassemble x."""
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2106_04756_b200 import instances, shard


def _csc(lp):
    a = sp.csr_matrix((lp.row_values, lp.row_cols, lp.row_start),
                      shape=(lp.num_rows, lp.num_cols))
    c = a.tocsc()
    c.sort_indices()
    return a, c


@pytest.mark.parametrize("cfg,scale", [(1, 1.0), (2, 0.002), (3, 0.0002), (5, 0.002)])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_rows_partition(cfg, scale, world):
    lp = instances.generate(cfg, 1, scale)
    b = shard.shard_rows(lp.num_rows, lp.row_start, world)
    assert b[0] == 0 and b[-1] == lp.num_rows
    assert np.all(np.diff(b) >= 0)
    # balanced on nonzeros + rows up to one row's weight
    w = lp.row_start[b[1:]] - lp.row_start[b[:-1]] + np.diff(b)
    heaviest_row = int(np.max(np.diff(lp.row_start))) + 1
    assert np.max(w) - np.min(w) <= 2 * heaviest_row + 1


@pytest.mark.parametrize("world", [2, 3])
def test_local_csc_partitions_the_entries(world):
    lp = instances.generate(2, 1, 0.002)
    a, c = _csc(lp)
    b = shard.shard_rows(lp.num_rows, lp.row_start, world)
    seen = np.zeros(a.nnz, dtype=np.int64)
    for r in range(world):
        lptr, pos = shard.local_csc(lp.num_cols, c.indptr, c.indices, b[r], b[r + 1])
        assert lptr[0] == 0 and lptr[-1] == len(pos)
        rows = c.indices[pos]
        assert np.all((rows >= b[r]) & (rows < b[r + 1]))
        # column j's local entries are a sub-range of full column j, in order
        for j in range(0, lp.num_cols, max(1, lp.num_cols // 50)):
            p = pos[lptr[j]:lptr[j + 1]]
            assert np.all((p >= c.indptr[j]) & (p < c.indptr[j + 1]))
            assert np.all(np.diff(p) == 1)
        seen[pos] += 1
    assert np.all(seen == 1)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("cfg,scale", [(2, 0.002), (5, 0.002)])
def test_local_csr_partitions_the_entries(cfg, scale, world):
    lp = instances.generate(cfg, 1, scale)
    a, c = _csc(lp)
    b = shard.shard_rows(lp.num_cols, c.indptr, world)  # column ranges
    assert b[0] == 0 and b[-1] == lp.num_cols
    seen = np.zeros(a.nnz, dtype=np.int64)
    for r in range(world):
        lptr, pos = shard.local_csr(lp.num_rows, c.indptr, c.indices, b[r], b[r + 1])
        assert lptr[0] == 0 and lptr[-1] == len(pos)
        assert np.all((pos >= c.indptr[b[r]]) & (pos < c.indptr[b[r + 1]]))
        rows = c.indices[pos]
        want = np.repeat(np.arange(lp.num_rows), np.diff(lptr))
        assert np.array_equal(rows, want)  # grouped by row
        cols = np.searchsorted(c.indptr, pos, side="right") - 1
        for i in range(0, lp.num_rows, max(1, lp.num_rows // 50)):
            assert np.all(np.diff(cols[lptr[i]:lptr[i + 1]]) > 0)  # columns ascend
        seen[pos] += 1
    assert np.all(seen == 1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank_main(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lp = instances.generate(2, 3, 0.003)
        a, c = _csc(lp)
        rng = np.random.default_rng(7)
        x = rng.standard_normal(lp.num_cols)
        y = rng.standard_normal(lp.num_rows)
        b = shard.shard_rows(lp.num_rows, lp.row_start, world)
        r0, r1 = int(b[rank]), int(b[rank + 1])
        lptr, pos = shard.local_csc(lp.num_cols, c.indptr, c.indices, r0, r1)
        # partial K'_p y_p from the shard's own entries and its own dual rows
        vals, rows = c.data[pos], c.indices[pos]
        part = np.zeros(lp.num_cols)
        cols = np.repeat(np.arange(lp.num_cols), np.diff(lptr))
        np.add.at(part, cols, vals * y[rows])
        t = torch.from_numpy(part)
        dist.all_reduce(t)
        kty_err = float(np.max(np.abs(t.numpy() - a.T @ y)) / (1 + np.max(np.abs(a.T @ y))))
        # K_p x over the shard's rows, reassembled by per-shard broadcasts
        kx = np.zeros(lp.num_rows)
        kx[r0:r1] = a[r0:r1] @ x
        full = torch.from_numpy(kx)
        for src in range(world):
            seg = full[int(b[src]):int(b[src + 1])].clone()
            dist.broadcast(seg, src=src)
            full[int(b[src]):int(b[src + 1])] = seg
        kx_exact = bool(np.array_equal(full.numpy(), a @ x))
        # identical decisions need identical sums on every shard
        s = torch.tensor([float(np.sum(part))])
        dist.all_reduce(s)
        gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, s.double())
        same = all(float(g) == float(gathered[0]) for g in gathered)
        # column partition: partial K_p x_p over the own columns, all-reduced
        bc = shard.shard_rows(lp.num_cols, c.indptr, world)
        c0, c1 = int(bc[rank]), int(bc[rank + 1])
        lptr, pos = shard.local_csr(lp.num_rows, c.indptr, c.indices, c0, c1)
        cols = np.searchsorted(c.indptr, pos, side="right") - 1
        rows = np.repeat(np.arange(lp.num_rows), np.diff(lptr))
        kxp = np.zeros(lp.num_rows)
        np.add.at(kxp, rows, c.data[pos] * x[cols])
        # peer exchange (FOLP_SHARD_EXCHANGE=peer): the partial lands in slot
        # `rank` of every rank's receive area, each rank sums its slots in
        # rank order -- identical sums everywhere without a data collective
        area = [torch.zeros(lp.num_rows, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(area, torch.from_numpy(kxp.copy()))
        peer = area[0].clone()
        for r in range(1, world):
            peer += area[r]
        everyone = [torch.zeros(lp.num_rows, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(everyone, peer)
        peer_ok = all(torch.equal(e, everyone[0]) for e in everyone)
        peer_ok = peer_ok and float(np.max(np.abs(peer.numpy() - a @ x))) <= 1e-12 * (1 + np.max(np.abs(a @ x)))
        t = torch.from_numpy(kxp)
        dist.all_reduce(t)
        kx_ref = a @ x
        kx_err = float(np.max(np.abs(t.numpy() - kx_ref)) / (1 + np.max(np.abs(kx_ref))))
        # x blocks reassembled by per-shard broadcasts of the own columns
        xs = np.zeros(lp.num_cols)
        xs[c0:c1] = x[c0:c1]
        fx = torch.from_numpy(xs)
        for src in range(world):
            seg = fx[int(bc[src]):int(bc[src + 1])].clone()
            dist.broadcast(seg, src=src)
            fx[int(bc[src]):int(bc[src + 1])] = seg
        x_exact = bool(np.array_equal(fx.numpy(), x))
        out.put((rank, kty_err, kx_exact and x_exact and kx_err <= 1e-12 and peer_ok, same, r1 - r0))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange_algebra():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert [r[0] for r in res] == [0, 1]
    for _, kty_err, kx_exact, same, rows in res:
        assert kty_err <= 1e-12
        assert kx_exact
        assert same
        assert rows > 0


def _pdual_rank_main(rank, world, port, out):
    """The partitioned dual epilogue (engine OpShardDualOwn) restated with
    gloo collectives: owner-only partial rows (a reduce-scatter in rank
    order), the dual step on the own rows, y' to every rank (all-gather) and
    the three trial sums folded over the ranks in rank order."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lp = instances.generate(5, 2, 0.004)
        a, c = _csc(lp)
        m = lp.num_rows
        rng = np.random.default_rng(11)
        x1 = rng.random(lp.num_cols)          # trial primal
        y0 = rng.standard_normal(m)
        y0[:lp.num_inequality_rows] = np.abs(y0[:lp.num_inequality_rows])
        kx0 = a @ rng.random(lp.num_cols)     # previous Kx
        sigma = 0.37
        bc = shard.shard_rows(lp.num_cols, c.indptr, world)
        c0, c1 = int(bc[rank]), int(bc[rank + 1])
        lptr, pos = shard.local_csr(m, c.indptr, c.indices, c0, c1)
        cols = np.searchsorted(c.indptr, pos, side="right") - 1
        rows = np.repeat(np.arange(m), np.diff(lptr))
        part = np.zeros(m)
        np.add.at(part, rows, c.data[pos] * x1[cols])
        chunk = (m + world - 1) // world
        r0, r1 = min(m, rank * chunk), min(m, (rank + 1) * chunk)
        # owner-only stores: every rank's partial rows of [r0, r1) reach this rank
        slots = [torch.zeros(m, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(slots, torch.from_numpy(part))
        kx1 = slots[0][r0:r1].numpy().copy()
        for r in range(1, world):
            kx1 = kx1 + slots[r][r0:r1].numpy()
        # dual step on the own rows (solver.cpp:66-82)
        i = np.arange(r0, r1)
        v = y0[i] + sigma * (lp.right_hand_side[i] - (2.0 * kx1 - kx0[i]))
        ineq = i < lp.num_inequality_rows
        v[ineq] = np.maximum(v[ineq], 0.0)
        dy = v - y0[i]
        sums = torch.tensor([np.sum(dy * (kx0[i] - kx1)), np.sum(dy * dy)], dtype=torch.float64)
        allsums = [torch.zeros(2, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allsums, sums)
        tot = allsums[0].clone()
        for r in range(1, world):
            tot += allsums[r]
        # y' assembled on every rank
        ypart = torch.zeros(m, dtype=torch.float64)
        ypart[r0:r1] = torch.from_numpy(v)
        yall = [torch.zeros(m, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(yall, ypart)
        y1 = sum(yall).numpy()
        # the unpartitioned dual step
        kx1f = a @ x1
        vf = y0 + sigma * (lp.right_hand_side - (2.0 * kx1f - kx0))
        vf[:lp.num_inequality_rows] = np.maximum(vf[:lp.num_inequality_rows], 0.0)
        dyf = vf - y0
        want = np.array([np.sum(dyf * (kx0 - kx1f)), np.sum(dyf * dyf)])
        scale = 1.0 + np.max(np.abs(vf))
        out.put((rank, float(np.max(np.abs(y1 - vf)) / scale),
                 float(np.max(np.abs(tot.numpy() - want) / (1.0 + np.abs(want)))),
                 tot.numpy().tolist(), r1 - r0))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_partitioned_dual_epilogue():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pdual_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert [r[0] for r in res] == [0, 1]
    assert res[0][3] == res[1][3]  # identical folded sums on both ranks
    for _, y_err, sum_err, _, rows in res:
        assert y_err <= 1e-13 and sum_err <= 1e-12 and rows > 0
