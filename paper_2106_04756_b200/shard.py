"""Multi-GPU row-sharded folp::solve (BASELINE.json north_star:
"K is row-partitioned across the 8 GPUs of one box, with NCCL over NVLink
... a reduce-scatter/allreduce of the partial K'y and the scalar
reductions").

One process per GPU under torch.distributed (the plumbing: rank, world and
the exchange of the NCCL unique id); the collectives themselves are NCCL
calls issued by the engine on its own stream (include/folp_gpu.h,
folp_gpu_shard).  Every rank calls `solve` with the same LP and parameters
and gets the same result.

`solve_loopback` runs `world` shards as host threads of this process on one
GPU through the engine's in-process loopback group -- the parity vehicle for
the sharded schedule when only one GPU is available.
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import Optional

import numpy as np

from . import cabi, engine


def _gpu_lib():
    return engine().lib


def _check(code: int) -> None:
    if code != cabi.FOLP_OK:
        lib = _gpu_lib()
        lib.folp_gpu_last_error.restype = C.c_char_p
        raise cabi.FolpError(code, lib.folp_gpu_last_error().decode(errors="replace"))


def shard_rows(m: int, row_start: np.ndarray, world: int) -> np.ndarray:
    """Row ranges [bounds[r], bounds[r+1]) of the shards (folp_gpu_shard_rows)."""
    rs = np.ascontiguousarray(row_start, dtype=np.int64)
    out = np.zeros(world + 1, dtype=np.int64)
    b = engine()
    _check(b.lib.folp_gpu_shard_rows(C.c_int64(m), rs.ctypes.data_as(C.POINTER(C.c_int64)),
                                      C.c_int32(world), out.ctypes.data_as(C.POINTER(C.c_int64))))
    return out


def local_csc(n: int, col_start: np.ndarray, col_rows: np.ndarray, r0: int, r1: int):
    """(lptr [n+1], pos [lnnz]): the CSC entries of rows [r0, r1) and their
    positions in the full CSC (folp_gpu_shard_local_csc)."""
    cs = np.ascontiguousarray(col_start, dtype=np.int64)
    cr = np.ascontiguousarray(col_rows, dtype=np.int64)
    lptr = np.zeros(n + 1, dtype=np.int64)
    pos = np.zeros(max(1, len(cr)), dtype=np.int64)
    lnnz = C.c_int64()
    b = engine()
    p64 = C.POINTER(C.c_int64)
    _check(b.lib.folp_gpu_shard_local_csc(
        C.c_int64(n), cs.ctypes.data_as(p64), cr.ctypes.data_as(p64), C.c_int64(r0),
        C.c_int64(r1), lptr.ctypes.data_as(p64), pos.ctypes.data_as(p64),
        C.c_int64(len(pos)), C.byref(lnnz)))
    return lptr, pos[:lnnz.value].copy()


def local_csr(m: int, col_start: np.ndarray, col_rows: np.ndarray, c0: int, c1: int):
    """(lptr [m+1], pos [lnnz]): the CSC entries of columns [c0, c1) in CSR
    order and their positions in the full CSC (folp_gpu_shard_local_csr)."""
    cs = np.ascontiguousarray(col_start, dtype=np.int64)
    cr = np.ascontiguousarray(col_rows, dtype=np.int64)
    lptr = np.zeros(m + 1, dtype=np.int64)
    pos = np.zeros(max(1, len(cr)), dtype=np.int64)
    lnnz = C.c_int64()
    b = engine()
    p64 = C.POINTER(C.c_int64)
    _check(b.lib.folp_gpu_shard_local_csr(
        C.c_int64(m), cs.ctypes.data_as(p64), cr.ctypes.data_as(p64), C.c_int64(c0),
        C.c_int64(c1), lptr.ctypes.data_as(p64), pos.ctypes.data_as(p64),
        C.c_int64(len(pos)), C.byref(lnnz)))
    return lptr, pos[:lnnz.value].copy()


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    b = engine()
    _check(b.lib.folp_gpu_nccl_unique_id(buf))
    return bytes(buf)


def nccl_spec(group=None, partition: str = "rows") -> cabi.ShardC:
    """Shard spec of this rank: rank 0 creates the NCCL unique id, every rank
    receives it through torch.distributed (any backend).  partition: "rows"
    (north_star: exchange n + 3 doubles per trial), "cols" (m + 2) or "auto"
    (the shorter exchange)."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        rank, world, obj = 0, 1, [nccl_unique_id()]  # a one-rank communicator
    else:
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
    spec = cabi.ShardC()
    spec.rank, spec.world, spec.backend = rank, world, cabi.SHARD_NCCL
    spec.partition = cabi.PARTITIONS[partition]
    C.memmove(spec.nccl_id, obj[0], 128)
    return spec


def solve(lp: cabi.LP, p: Optional[dict] = None, x0=None, y0=None, group=None,
          partition: str = "rows", **kw):
    """folp::solve as this rank's shard (torch.distributed initialized,
    one process per GPU, FOLP_DEVICE / cuda current device = this rank's GPU)."""
    return engine().solve_lp(lp, p, x0, y0, shard=nccl_spec(group, partition), **kw)


class LoopbackGroup:
    def __init__(self, world: int):
        b = engine()
        h = C.c_void_p()
        b.lib.folp_gpu_loopback_create.argtypes = [C.c_int32, C.POINTER(C.c_void_p)]
        _check(b.lib.folp_gpu_loopback_create(C.c_int32(world), C.byref(h)))
        self.h, self.world = h, world

    def spec(self, rank: int, partition: str = "rows") -> cabi.ShardC:
        s = cabi.ShardC()
        s.rank, s.world, s.backend, s.loopback = rank, self.world, cabi.SHARD_LOOPBACK, self.h
        s.partition = cabi.PARTITIONS[partition]
        return s

    def close(self):
        if self.h:
            lib = _gpu_lib()
            lib.folp_gpu_loopback_destroy.argtypes = [C.c_void_p]
            lib.folp_gpu_loopback_destroy(self.h)
            self.h = None


def solve_loopback(lp: cabi.LP, world: int, p: Optional[dict] = None,
                   partition: str = "rows", **kw) -> list:
    """`world` shards as threads of this process on one GPU; returns the
    per-shard results (they must be identical)."""
    g = LoopbackGroup(world)
    out: list = [None] * world
    errs: list = [None] * world

    def run(r):
        try:
            out[r] = engine().solve_lp(lp, p, shard=g.spec(r, partition), **kw)
        except BaseException as e:  # noqa: BLE001 -- re-raised below
            errs[r] = e

    try:
        threads = [threading.Thread(target=run, args=(r,)) for r in range(world)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    finally:
        g.close()
    for e in errs:
        if e is not None:
            raise e
    return out
