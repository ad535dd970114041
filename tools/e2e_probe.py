"""Per-step wall times of the cfg2 e2e path (ingest_simulation from pinned host
columns), to look at the spread behind bench.py's e2e number.
python tools/e2e_probe.py [steps]; STROM_H2D_RING / STROM_H2D_CHUNK apply."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1910_01260_b200 import _capi, basis, workloads as wl  # noqa: E402

def pool_reserved():
    """Bytes reserved by the device's default stream-ordered pool (the library's allocator)."""
    from cuda.bindings import runtime as rt

    _, pool = rt.cudaDeviceGetDefaultMemPool(torch.cuda.current_device())
    _, v = rt.cudaMemPoolGetAttribute(pool, rt.cudaMemPoolAttr.cudaMemPoolAttrReservedMemCurrent)
    return int(v)


steps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
xt, _, _, _ = wl.cfg2_stream_torch(n=bench.N_S, cols=bench.COLS, rank=bench.RANK, seed=0, device=torch.device("cuda"))
st0 = basis.isvd_init(xt[0], bench.TOL, tol_sv=bench.TOL, r_max=bench.RANK, cap_mode="truncate")
st100 = basis.ingest_simulation(st0, xt[1:bench.WARM_COLS].T)
host = torch.empty((bench.COLS - bench.WARM_COLS, bench.N_S), dtype=torch.float64, pin_memory=True)
host.copy_(xt[bench.WARM_COLS:])
cols_h = host.T
dcols = xt[bench.WARM_COLS:].T
prof = len(sys.argv) > 2 and sys.argv[2] == "prof"
# heartbeat thread: gaps in it mean the whole process stalled (OS), not one API call
import threading  # noqa: E402

beats = []
stop_beat = threading.Event()


def heartbeat():
    while not stop_beat.is_set():
        beats.append(time.perf_counter())
        time.sleep(0.001)


threading.Thread(target=heartbeat, daemon=True).start()
for name, src in (("device", dcols), ("host", cols_h), ("device", dcols), ("host", cols_h)):
    ts, gs, hs, pool, kms, starts = [], [], [], [], [], []
    for _ in range(steps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        starts.append(t0)
        e0.record()
        if prof:
            _capi.lib.strom_profile_reset()
            _capi.lib.strom_profile_enable(1)
        s = basis.ingest_simulation(st100, src)
        t1 = time.perf_counter()
        e1.record()
        s.sigma.cpu()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
        hs.append(1e3 * (t1 - t0))
        gs.append(e0.elapsed_time(e1))
        pool.append(pool_reserved() / 1e9)
        if prof:
            _capi.lib.strom_profile_enable(0)
            pms = (_capi.dbl * 16)()
            _capi.lib.strom_profile_read(16, None, pms, None)
            kms.append([round(pms[k], 1) for k in range(len(bench.PROF_KINDS))])
    print(name, "wall", " ".join(f"{t:.1f}" for t in ts), flush=True)
    print(name, "call", " ".join(f"{t:.1f}" for t in hs), flush=True)
    print(name, "pool GB", " ".join(f"{x:.1f}" for x in pool), flush=True)
    for i in range(len(ts)):
        if ts[i] > 1.5 * min(ts):
            t_end = starts[i] + ts[i] / 1e3
            bb = [b for b in beats if starts[i] <= b <= t_end]
            gaps = sorted((b - a for a, b in zip(bb, bb[1:])), reverse=True)[:3]
            print(name, "outlier step", i, f"{ts[i]:.1f} ms; largest heartbeat gaps (ms)",
                  [round(1e3 * g, 1) for g in gaps], flush=True)
    for i, row in enumerate(kms):
        if ts[i] > 1.2 * min(ts):
            print(name, "slow step", i, f"{ts[i]:.1f} ms, kernel ms by kind", dict(zip(bench.PROF_KINDS, row)), flush=True)
    print(name, "evts", " ".join(f"{t:.1f}" for t in gs), "ms; rank", s.rank, flush=True)
