"""Row-sharded incremental SVD (csrc/shard.cuh) on ONE GPU.

The multi-GPU exchange cannot run on a one-GPU box with kernels of different
ranks waiting on each other, so two harnesses cover it:

* world = 1 through the production path (IPC mailbox set-up minus the peers,
  the single flag kernel): the exchange degenerates to a copy through the
  mailbox and the result must be BIT-identical to the unsharded state;
* world = 2 / 3 as a single-process group (ShardGroup.local): each virtual
  rank owns its row block and runs on its own host thread and stream; the
  publish and combine halves of the exchange kernel are ordered by stream
  events.  The replicated state must be bit-identical across the ranks, agree
  with the unsharded device run to rounding, and with the CPU oracle
  (reference basis.py:105-194) on the same snapshots.
"""

import threading

import numpy as np
import pytest
import torch

from oracle import strom_oracle as so
from paper_1910_01260_b200 import basis, workloads as wl
from paper_1910_01260_b200.sharded import ShardGroup, partition_rows

from helpers import npy, principal_sine

pytestmark = pytest.mark.gpu


def run_ranks(world, fn, timeout=600):
    """fn(rank) on one host thread and one CUDA stream per virtual rank."""
    res, err = [None] * world, [None] * world

    def target(r):
        try:
            torch.cuda.set_device(0)
            with torch.cuda.stream(torch.cuda.Stream()):
                res[r] = fn(r)
                torch.cuda.current_stream().synchronize()
        except BaseException as e:  # noqa: BLE001 -- reported by the caller
            err[r] = e

    ts = [threading.Thread(target=target, args=(r,), daemon=True) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout)
        assert not t.is_alive(), "a virtual rank hung"
    for e in err:
        if e is not None:
            raise e
    return res


def sharded_stream(groups, x, tol, updates_one_by_one=0, splits=(), **kw):
    """Every rank: isvd_init on column 0, `updates_one_by_one` single updates, then
    ingest_simulation over the rest (in the given column splits).  Returns per rank
    (phi_local, sigma, v, counters, exchanges)."""
    xd = torch.as_tensor(x, device="cuda")
    ncols = x.shape[1]

    def body(r):
        g = groups[r]
        xl = g.rows(xd).contiguous()
        with g:
            st = basis.isvd_init(xl[:, 0].contiguous(), tol, **kw)
        j = 1
        for _ in range(updates_one_by_one):
            st = basis.isvd_update(st, xl[:, j].contiguous())
            j += 1
        for end in list(splits) + [ncols]:
            if end > j:
                st = basis.ingest_simulation(st, xl[:, j:end])
                j = end
        out = (npy(st.phi), npy(st.sigma), npy(st.v),
               (st.n_rejected, st.n_dependent, st.n_truncated, st.n_restarts), g.status())
        return out

    return run_ranks(len(groups), body)


def unsharded_stream(x, tol, updates_one_by_one=0, splits=(), **kw):
    xd = torch.as_tensor(x, device="cuda")
    st = basis.isvd_init(xd[:, 0].contiguous(), tol, **kw)
    j = 1
    for _ in range(updates_one_by_one):
        st = basis.isvd_update(st, xd[:, j].contiguous())
        j += 1
    for end in list(splits) + [x.shape[1]]:
        if end > j:
            st = basis.ingest_simulation(st, xd[:, j:end])
            j = end
    return npy(st.phi), npy(st.sigma), npy(st.v), (st.n_rejected, st.n_dependent, st.n_truncated, st.n_restarts)


def lowrank(n, cols, rank, seed, decades_per=4.0):
    x, _, _, _ = wl.cfg2_stream_numpy(n=n, cols=cols, rank=rank, seed=seed, decades_per=decades_per)
    return np.ascontiguousarray(x)


def test_partition_rows():
    assert partition_rows(1 << 20, 2, 1) == (1 << 19, 1 << 19)
    assert partition_rows(1000, 3, 0) == (0, 384)
    assert partition_rows(1000, 3, 2) == (768, 232)
    with pytest.raises(ValueError):
        partition_rows(200, 3, 2)  # the third block would be empty


def test_world1_flag_kernel_is_bit_identical(cuda):
    """Production path, one rank: mailbox create / connect, the single exchange
    kernel with its release / acquire flags; a copy through the mailbox."""
    n, cols = 4096, 60
    x = lowrank(n, cols, 12, seed=3)
    ref = unsharded_stream(x, 1e-10, updates_one_by_one=3, tol_sv=1e-12, r_max=16, cap_mode="truncate")
    g = ShardGroup.connect(n)
    assert (g.rank, g.world, g.row0, g.n_local) == (0, 1, 0, n)
    got = sharded_stream([g], x, 1e-10, updates_one_by_one=3, tol_sv=1e-12, r_max=16, cap_mode="truncate")[0]
    assert got[3] == ref[3]
    np.testing.assert_array_equal(got[1], ref[1])
    np.testing.assert_array_equal(got[2], ref[2])
    np.testing.assert_array_equal(got[0], ref[0])
    exchanges, err = got[4]
    assert err == 0 and exchanges >= cols // 8  # at least every window pass crossed the mailbox


@pytest.mark.parametrize("world,n", [(2, 8192), (3, 5000)])
def test_virtual_ranks_match_unsharded_and_oracle(cuda, world, n):
    cols, rank, tol = 72, 8, 1e-9
    x, _, _, _ = wl.cfg2_stream_numpy(n=n, cols=cols, rank=rank, seed=11, noise=1e-7, decades_per=4.0)
    x = np.ascontiguousarray(x)
    # noise well above tol: every snapshot is independent and truncated at the cap,
    # the store gains a column per update and is compacted (a Gram exchange) every
    # ~16 updates
    kw = dict(tol_sv=0.0, r_max=12, cap_mode="truncate")
    ref = unsharded_stream(x, tol, updates_one_by_one=2, **kw)
    assert ref[3][2] >= 40
    groups = ShardGroup.local(world, n)
    outs = sharded_stream(groups, x, tol, updates_one_by_one=2, **kw)
    # replicated state: bit-identical on every rank
    for o in outs[1:]:
        np.testing.assert_array_equal(o[1], outs[0][1])
        np.testing.assert_array_equal(o[2], outs[0][2])
        assert o[3] == outs[0][3]
        assert o[4] == outs[0][4] and o[4][1] == 0
    # the row blocks tile phi
    phi = np.vstack([o[0] for o in outs])
    assert phi.shape[0] == n
    sig = outs[0][1]
    # against the unsharded device run: the same algorithm with another summation
    # split; the signal modes agree to rounding (noise-level modes follow decisions)
    m = rank
    assert np.max(np.abs(sig[:m] - ref[1][:m]) / ref[1][:m]) <= 1e-11
    assert principal_sine(phi[:, :m - 2], ref[0][:, :m - 2]) <= 1e-8
    # against the oracle (the reference's algorithm) on the same snapshots
    o = so.stream(x, tol, **kw)
    assert np.max(np.abs(sig[:m] - o.sigma[:m]) / o.sigma[:m]) <= 1e-10
    assert principal_sine(phi[:, :m - 2], o.phi[:, :m - 2]) <= 1e-8
    # phi = U W is orthonormal to the representation's defect
    assert np.max(np.abs(phi[:, :m].T @ phi[:, :m] - np.eye(m))) <= 1e-8
    # and V with it: X ~ phi diag(sigma) V^T on the signal part
    recon = phi @ np.diag(sig) @ outs[0][2].T
    assert np.max(np.abs(recon - x)) <= 1e-4 * np.max(np.abs(x))  # the truncated noise


def test_virtual_ranks_per_snapshot_pipeline(cuda):
    """A capped stream of independent snapshots: after 64 truncations without a
    dependent update ingest_simulation takes the per-snapshot fused pipeline
    (the cfg5 case, the one row sharding is for)."""
    n, cols, cap = 4096, 120, 6
    rng = np.random.default_rng(5)
    q, _ = np.linalg.qr(rng.standard_normal((n, 4)))
    x = q @ (rng.standard_normal((4, cols)) * np.array([1.0, 0.3, 0.1, 0.03])[:, None])
    x = np.ascontiguousarray(x + 1e-4 * rng.standard_normal((n, cols)))  # every snapshot independent
    kw = dict(tol_sv=0.0, r_max=cap, cap_mode="truncate")
    splits = (90,)  # the second call starts after >= 64 truncations
    ref = unsharded_stream(x, 1e-9, splits=splits, **kw)
    assert ref[3][1] == 0 and ref[3][2] >= 64  # no dependent update, rank cap hit throughout
    groups = ShardGroup.local(2, n)
    outs = sharded_stream(groups, x, 1e-9, splits=splits, **kw)
    np.testing.assert_array_equal(outs[0][1], outs[1][1])
    np.testing.assert_array_equal(outs[0][2], outs[1][2])
    assert outs[0][3] == ref[3] and outs[0][4][1] == 0
    sig = outs[0][1]
    assert np.max(np.abs(sig[:4] - ref[1][:4]) / ref[1][:4]) <= 1e-10
    o = so.stream(x, 1e-9, **kw)
    assert np.max(np.abs(sig[:3] - o.sigma[:3]) / o.sigma[:3]) <= 1e-8  # a truncating stream: leading modes


def test_diverging_ranks_fail_instead_of_hanging(cuda, monkeypatch):
    """A peer that never publishes makes the flag kernel time out and the state
    report it; the GPU is never left spinning."""
    import ctypes as C

    from paper_1910_01260_b200 import _capi as capi

    monkeypatch.setenv("STROM_SHARD_TIMEOUT_MS", "200")
    # a two-rank flag-mode group whose peer is this process's second mailbox, never driven
    out0, out1 = C.c_void_p(), C.c_void_p()
    h0, h1 = (C.c_char * 64)(), (C.c_char * 64)()
    capi.call("strom_shard_mailbox_create", 2, C.byref(out0), h0)
    capi.call("strom_shard_mailbox_create", 2, C.byref(out1), h1)
    try:
        # the same process cannot open its own IPC handle: connect must refuse cleanly or work;
        # either way nothing may hang
        rc = capi.lib.strom_shard_connect(out0, 0, 1024, bytes(h0.raw) + bytes(h1.raw))
        if rc != 0:
            assert "cudaIpcOpenMemHandle" in capi.last_error()
            return
        g = ShardGroup(out0.value, 0, 2, 1024)
        out0 = C.c_void_p()  # owned by g now
        x = torch.randn(512, dtype=torch.float64, device="cuda")
        with g:
            st = basis.isvd_init(x, 1e-8)
        with pytest.raises(RuntimeError, match="timed out"):
            st.rank
    finally:
        for o in (out0, out1):
            if o.value:
                capi.lib.strom_shard_free(o)
        # a refused connect or a timed-out exchange must not leave a CUDA error behind
        # for the next launch check of an unrelated call
        y = torch.randn(256, 3, dtype=torch.float64, device="cuda")
        st2 = basis.ingest_simulation(basis.isvd_init(y[:, 0].contiguous(), 1e-8), y[:, 1:])
        assert st2.rank == 3
        from paper_1910_01260_b200 import linalg
        q, r = linalg.qr(y)
        assert torch.allclose(q @ r, y, atol=1e-12)
