"""N>1 host logic of bench.py on CPU: world size 2 over gloo (127.0.0.1).

bench.py --gpus N runs N independent replicas of the cfg2 stream (DESIGN.md
section 6): no collective on the data path, only the barrier, the max-over-
ranks device time and the rank-0 JSON line.  These tests drive exactly those
helpers with the gloo backend.
"""
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, ws, port, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(ws), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench
    import torch.distributed as dist

    try:
        got_ws, got_rank, _ = bench.dist_setup(ws, backend="gloo")
        bench.barrier(got_ws)
        ms = 10.0 + 5.0 * rank  # rank 1 is the slow one
        ms_max = bench.allmax(got_ws, ms)
        rate = bench.whole_job_rate(400, 5, got_ws, ms_max)
        seed = bench.replica_seed(got_rank)
        bench.barrier(got_ws)
        q.put((rank, got_ws, got_rank, ms_max, rate, seed))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_replica_timing_world2_gloo():
    ws, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, got_ws, got_rank, ms_max, rate, seed in res:
        assert (got_ws, got_rank) == (ws, rank)
        assert ms_max == 15.0  # max over ranks, identical everywhere
        assert rate == pytest.approx(400 * 5 * 2 / 0.015)  # whole-job units / slowest rank
    assert {r[5] for r in res} == {0}  # every replica ingests the reference arm's stream (numpy seed 0)


def test_reference_arm_rank_gating(monkeypatch, capsys):
    """Under torchrun only rank 0 runs the reference arm; other ranks exit silently."""
    sys.path.insert(0, ROOT)
    import bench

    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")

    class A:
        steps, warmup = 1, 3

    assert bench.run_reference(A()) is None
    assert capsys.readouterr().out == ""


def test_reference_arm_never_maps_the_library():
    """The reference arm loads the numpy generators by path: neither the product
    package nor libstrom_b200.so may enter the process (BENCH native_so_loaded)."""
    import subprocess

    code = ("import sys; sys.path.insert(0, %r); import bench; wl = bench._workloads(); "
            "x, _, _, _ = wl.cfg2_stream_numpy(n=256, cols=8, rank=4); "
            "from oracle import strom_oracle; "
            "assert not any(m.startswith('paper_1910_01260_b200') for m in sys.modules), sorted(sys.modules); "
            "maps = open('/proc/self/maps').read(); assert 'libstrom_b200' not in maps; print('clean')" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    assert "clean" in out.stdout
