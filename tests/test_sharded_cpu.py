"""Row-sharded incremental SVD: the host side and the exchange
protocol on CPU, world size 2 over gloo (127.0.0.1).

The device exchange (csrc/shard.cuh) gives every rank every rank's partial sums
and adds them in RANK order, so the replicated small state (sigma, V, N, L, the
decisions) is bit-identical on all ranks.  Here the same protocol runs with the
NumPy model of the device algorithm (tests/device_model.py, `BlockSums`): each
gloo rank owns its row block (`partition_rows`), the partials travel by
`all_gather`, and

* the two ranks' replicated state must be equal bit for bit,
* equal bit for bit to the same two row blocks driven inside ONE process
  (two threads, partials handed over in memory) -- the transport adds nothing,
* and agree with the unsharded model and with the oracle (the reference's
  algorithm, basis.py:105-194) to rounding.

`gather_handles` (the mailbox-handle all-gather `ShardGroup.connect` performs)
is driven with gloo as well.
"""
import os
import socket
import sys
import threading

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

N, COLS, RANK, TOL = 1000, 40, 6, 1e-9
KW = dict(tol_sv=0.0, r_max=8, ccap=13)  # an append per update: a compaction (Gram exchange) every ~4


def _stream():
    rng = np.random.default_rng(21)
    q, _ = np.linalg.qr(rng.standard_normal((N, RANK)))
    w = rng.standard_normal((RANK, COLS)) * (10.0 ** (-np.arange(RANK) / 2.0))[:, None]
    return np.ascontiguousarray(q @ w + 1e-6 * rng.standard_normal((N, COLS)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _partition(n, world, rank):
    # sharded.py imports the ctypes binding at module import; load it by path with a stub
    # so the CPU suite never needs the CUDA library for the host-side arithmetic
    import importlib.util
    import types

    pkg = types.ModuleType("_shard_stub_pkg")
    pkg.__path__ = []
    sys.modules.setdefault("_shard_stub_pkg", pkg)
    sys.modules.setdefault("_shard_stub_pkg._capi", types.ModuleType("_shard_stub_pkg._capi"))
    spec = importlib.util.spec_from_file_location(
        "_shard_stub_pkg.sharded", os.path.join(ROOT, "paper_1910_01260_b200", "sharded.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod, mod.partition_rows(n, world, rank)


def _run_model(x_local, exchange):
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    sys.path.insert(0, ROOT)
    import device_model as dm

    s = dm.init(x_local[:, 0], TOL, n=N, sums=dm.BlockSums(exchange), **KW)
    flags = []
    for j in range(1, x_local.shape[1]):
        s = dm.update(s, x_local[:, j])
        flags.append((s.flags["dep"], s.flags["trunc"], s.flags["qr"], s.flags["appended"]))
    return s, flags


def _worker(rank, ws, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(ws), MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        mod, (row0, nloc) = _partition(N, ws, rank)
        # the handle all-gather of ShardGroup.connect
        mine = bytes([rank * 16 + i % 16 for i in range(mod.HANDLE_BYTES)])
        handles = mod.gather_handles(mine, ws, None, torch.device("cpu"))
        n_exch = [0]

        def exchange(partial):
            n_exch[0] += 1
            t = torch.from_numpy(np.ascontiguousarray(partial).reshape(-1).copy())
            outs = [torch.empty_like(t) for _ in range(ws)]
            dist.all_gather(outs, t)
            return [o.numpy().reshape(partial.shape) for o in outs]

        x = _stream()[row0:row0 + nloc]
        s, flags = _run_model(x, exchange)
        dist.barrier()
        q.put((rank, row0, nloc, handles, s.sigma.tobytes(), s.V.tobytes(), s.W.tobytes(), s.L.tobytes(),
               flags, n_exch[0], s.phi.copy()))
    finally:
        dist.destroy_process_group()


def _in_process(ws):
    """The same row blocks on `ws` threads of one process, partials handed over in memory."""
    x = _stream()
    box, bar = [None] * ws, threading.Barrier(ws)
    out = [None] * ws

    def body(r):
        _, (row0, nloc) = _partition(N, ws, r)

        def exchange(partial):
            box[r] = np.array(partial, dtype=float, copy=True)
            bar.wait()
            parts = [box[p].copy() for p in range(ws)]
            bar.wait()
            return parts

        out[r] = _run_model(x[row0:row0 + nloc], exchange)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(ws)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(300)
    return out


def test_partition_rows_cpu():
    mod, got = _partition(1 << 20, 2, 1)
    assert got == (1 << 19, 1 << 19)
    assert mod.partition_rows(1000, 3, 0) == (0, 384)
    assert mod.partition_rows(1000, 3, 2) == (768, 232)
    assert mod.partition_rows(1 << 26, 8, 7) == (7 << 23, 1 << 23)
    # the blocks tile [0, n) without gaps, starting on store-tile boundaries
    for n, w in ((1000, 2), (5000, 3), (12345, 8)):
        at = 0
        for r in range(w):
            r0, nl = mod.partition_rows(n, w, r)
            assert r0 == at and r0 % mod.ROW_ALIGN == 0 and nl > 0
            at += nl
        assert at == n
    with pytest.raises(ValueError):
        mod.partition_rows(200, 3, 2)  # the third block would be empty
    with pytest.raises(ValueError):
        mod.partition_rows(1000, 9, 0)
    with pytest.raises(ValueError):
        mod.partition_rows(1000, 2, 2)


def test_two_rank_update_is_bit_identical_world2_gloo():
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted((q.get(timeout=240) for _ in range(ws)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = res
    # row blocks tile the matrix; the handles arrive in rank order on both ranks
    assert (a[1], a[2], b[1], b[2]) == (0, 512, 512, 488)
    assert a[3] == b[3] and len(a[3]) == 128 and a[3][0] == 0 and a[3][64] == 16
    # replicated state and decisions: the same bits on both ranks
    for k in (4, 5, 6, 7):
        assert a[k] == b[k]
    assert a[8] == b[8] and a[9] == b[9] and a[9] >= COLS  # >= one exchange per update
    assert any(f[3] for f in a[8]) and any(f[1] for f in a[8])  # appends and truncations occurred

    # the same blocks inside one process: the transport changes nothing
    loc = _in_process(ws)
    s0, flags0 = loc[0]
    assert s0.sigma.tobytes() == a[4] and s0.V.tobytes() == a[5]
    assert s0.W.tobytes() == a[6] and s0.L.tobytes() == a[7]
    assert flags0 == a[8]
    assert loc[1][0].sigma.tobytes() == a[4]
    np.testing.assert_array_equal(np.vstack([loc[0][0].phi, loc[1][0].phi]), np.vstack([a[10], b[10]]))

    # against the unsharded model and the oracle: another summation split, same algorithm
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import device_model as dm
    from oracle import strom_oracle as so

    x = _stream()
    one = dm.stream(x, TOL, **KW)
    sig = np.frombuffer(a[4])
    m = RANK
    assert np.max(np.abs(sig[:m] - one.sigma[:m]) / one.sigma[:m]) <= 1e-11
    o = so.stream(x, TOL, tol_sv=0.0, r_max=8, cap_mode="truncate")
    assert np.max(np.abs(sig[:m] - o.sigma[:m]) / o.sigma[:m]) <= 1e-9
    phi = np.vstack([a[10], b[10]])
    sv = np.linalg.svd(phi[:, :m - 1].T @ o.phi[:, :m - 1], compute_uv=False)
    assert np.sqrt(max(0.0, 1.0 - sv.min() ** 2)) <= 1e-6
