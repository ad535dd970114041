"""Row-sharded incremental SVD over the GPUs of one NVSwitch domain.

The reference's iSVD (basis.py:105-194) is single-process.  Its tall work is
row-local -- the projection and the Pythagorean residual (basis.py:135-139) and
the new direction (basis.py:150-156) are sums over rows -- so rank ``r`` of a
group owns a contiguous block of rows of every snapshot and of the left basis,
while sigma, V and every decision are replicated bit-identically.  The per-rank
partial sums cross the GPUs in one small kernel over NVLink peer memory
(``csrc/shard.cuh``), summed in rank order on every rank.

Usage, one process per GPU under ``torch.distributed``::

    group = ShardGroup.connect(n_global)            # collective
    x_loc = group.rows(x0)                          # this rank's rows
    with group:
        state = basis.isvd_init(x_loc, tol)         # the rank's shard of the state
    state = basis.ingest_simulation(state, group.rows(X))
    state.sigma, state.v                            # replicated
    state.phi                                       # rows [group.row0, group.row0 + group.n_local)

Every rank must issue the same sequence of calls.  ``ShardGroup.local`` builds
``world`` virtual ranks inside one process for the one-GPU tests (one host
thread per rank; stream events order the exchanges).
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _capi as capi

HANDLE_BYTES = 64
MAX_RANKS = 8
ROW_ALIGN = 128  # row blocks start on a store-tile boundary (ldu = round_up(n, 128))

__all__ = ["ShardGroup", "partition_rows", "gather_handles"]


def partition_rows(n_global: int, world: int, rank: int, align: int = ROW_ALIGN) -> tuple[int, int]:
    """(row0, n_local) of ``rank``: equal blocks of ceil(n / world) rows rounded
    up to ``align``; the last ranks take what is left (possibly fewer rows, never
    none unless n_global < world * align)."""
    if not (1 <= world <= MAX_RANKS):
        raise ValueError(f"shard groups hold 1..{MAX_RANKS} ranks, got {world}")
    if not (0 <= rank < world):
        raise ValueError(f"rank {rank} outside a group of {world}")
    if n_global < 1:
        raise ValueError("need n_global >= 1")
    per = -(-n_global // world)
    per = -(-per // align) * align
    row0 = min(rank * per, n_global)
    n_local = min(per, n_global - row0)
    if n_local <= 0:
        raise ValueError(f"rank {rank} of {world} owns no rows of {n_global} (blocks of {per})")
    return row0, n_local


def gather_handles(handle: bytes, world: int, pg=None, device=None) -> bytes:
    """All-gather the ranks' 64-byte mailbox handles in rank order over
    ``torch.distributed`` (any backend: the tensor lives on ``device``)."""
    import torch.distributed as dist

    if len(handle) != HANDLE_BYTES:
        raise ValueError(f"mailbox handles are {HANDLE_BYTES} bytes")
    if world == 1:
        return bytes(handle)
    mine = torch.tensor(list(handle), dtype=torch.uint8, device=device)
    outs = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(outs, mine, group=pg)
    return b"".join(bytes(t.cpu().tolist()) for t in outs)


class ShardGroup:
    """One rank's membership of a row-shard group (a ``strom_shard`` handle)."""

    def __init__(self, handle, rank: int, world: int, n_global: int, keep=None):
        self._h = handle
        self.rank, self.world, self.n_global = int(rank), int(world), int(n_global)
        self.row0, self.n_local = partition_rows(n_global, world, rank)
        self._keep = keep

    # -- construction ------------------------------------------------------
    @classmethod
    def connect(cls, n_global: int, pg=None) -> "ShardGroup":
        """Collective over ``pg`` (default: the world group): allocate this rank's
        mailbox on the current CUDA device, exchange the IPC handles, map the peers."""
        import torch.distributed as dist

        world = dist.get_world_size(pg) if dist.is_initialized() else 1
        rank = dist.get_rank(pg) if dist.is_initialized() else 0
        out = C.c_void_p()
        mine = (C.c_char * HANDLE_BYTES)()
        capi.call("strom_shard_mailbox_create", world, C.byref(out), mine)
        backend = dist.get_backend(pg) if world > 1 else "gloo"
        dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
        handles = gather_handles(bytes(mine.raw), world, pg, dev)
        capi.call("strom_shard_connect", out, rank, int(n_global), handles)
        if world > 1:
            dist.barrier(group=pg)  # every mailbox is mapped before anyone publishes
        return cls(out.value, rank, world, n_global)

    @classmethod
    def local(cls, world: int, n_global: int) -> list["ShardGroup"]:
        """``world`` virtual ranks in this process on the current device (tests)."""
        arr = (C.c_void_p * world)()
        capi.call("strom_shard_create_local", world, int(n_global), arr)
        return [cls(arr[r], r, world, n_global) for r in range(world)]

    # -- use ------------------------------------------------------------------
    def rows(self, x):
        """This rank's row block of a full-length vector or matrix (a view)."""
        if x.shape[0] != self.n_global:
            raise ValueError(f"expected {self.n_global} rows, got {x.shape[0]}")
        return x[self.row0:self.row0 + self.n_local]

    def __enter__(self):
        capi.lib.strom_shard_make_current(self._h)
        return self

    def __exit__(self, *exc):
        capi.lib.strom_shard_make_current(None)
        return False

    def status(self) -> tuple[int, int]:
        """(exchanges completed, sticky error word); synchronises the device."""
        n, err = C.c_int64(), C.c_int32()
        capi.call("strom_shard_status", self._h, C.byref(n), C.byref(err))
        return int(n.value), int(err.value)

    def close(self) -> None:
        h, self._h = self._h, None
        if h:
            capi.lib.strom_shard_free(h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass
