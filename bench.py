#!/usr/bin/env python
"""Benchmark of the B200 hot path on the BASELINE.json workloads.

Metric (BASELINE.json): "iSVD snapshots/s at n_s=1M fp64 (% HBM roofline);
ST-ROM operator build ms".

* Primary line (``value``): device iSVD ingestion on config 2 -- n_s = 2^20,
  the 500-snapshot stream X = Q diag(10^(-i/8)) W^T + 1e-12 E built with
  numpy ``default_rng(0)`` in SURVEY 8(d)'s draw order (Q, W, E), tol_svd =
  tol_sv = 1e-9, r_max = 64 (truncate).  Both arms start from the same state:
  the rank-64 truncated SVD of snapshots 1-100 (numpy QR + SVD, k = 100), and
  ingest the same bytes.  One step = ``ingest_simulation`` of snapshots
  101-500 with X resident in HBM; U (>= 512 MB) and X (4.2 GB) exceed L2, so
  no flush is needed.  value = snapshots/s over all ranks.
* ``seeds``: the same step on two more streams (torch generator seeds 1, 2,
  generated on the device) -- decision counts and rates, and the median over
  the three seeds, since throughput follows noise-level decisions.
* ``e2e``: the same step through the public API from pinned HOST memory
  (chunked H2D overlapped with the updates inside the C ABI) plus the D2H
  read of sigma; ``e2e_pageable`` from the numpy array itself.
* ``st_build``: config 4 operator build {A_hat, B_hat, x0_hat, A_st, f_st,
  x0_st} (N = 10^6, n_s = 50, n_t = 20, N_t = 500), ms per build, device
  resident and end to end from host CSR / Phi_s / Psi; the dense solve is
  reported separately.
* ``cfg1``, ``cfg3``, ``cfg5``: the other BASELINE configurations (whole cfg1
  pipeline; transport proxy; capacity run, bounded).
* ``cpu_baseline``: the CPU oracle port (numpy/OpenBLAS, all host cores) on a
  bounded sample of the same workloads, rank 0, N = 1.

``--impl reference`` times the oracle port of the reference (pure
Python/NumPy; the reference itself cannot travel to the GPU box, DESIGN.md
section 5) on the same cfg2 workload: same bytes, same starting state, each
step two consecutive updates from snapshot 101 on.  That arm never imports the
product package, so the sm_100a library is not mapped.
Multi-GPU (torchrun): independent replicas, one stream per rank.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

METRIC = "iSVD snapshots/s at n_s=1M fp64 (% HBM roofline); ST-ROM operator build ms"
N_S = 1 << 20
COLS = 500
WARM_COLS = 100
RANK = 64
TOL = 1e-9
PROF_KINDS = ["u_pass", "reorth_pass", "decide", "core_step", "v_update", "compact_prep", "compact_sweep",
              "spatial", "st_gemm", "st_small", "lu", "temporal", "other", "window_pass"]
WORKLOAD = ("cfg2: n_s=2^20 fp64, 500-snapshot stream X=Q diag(10^(-i/8)) W^T + 1e-12 N(0,1) from numpy "
            "default_rng(0) (draw order Q, W, E); tol_svd=tol_sv=1e-9, r_max=64 truncate; start = rank-64 "
            "truncated SVD of snapshots 1-100 (k=100); step = isvd_update over snapshots 101-500 in order")


def peaks():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _workloads():
    """paper_1910_01260_b200/workloads.py loaded by path: the generators are
    numpy/scipy only, and importing the package would map the sm_100a library
    (the reference arm must not)."""
    name = "strom_bench_workloads"
    if name in sys.modules:
        return sys.modules[name]
    spec = importlib.util.spec_from_file_location(name, os.path.join(HERE, "paper_1910_01260_b200", "workloads.py"))
    mod = importlib.util.module_from_spec(spec)
    sys.modules[name] = mod
    spec.loader.exec_module(mod)
    return mod


def cfg2_host():
    """The cfg2 stream (numpy seed 0, n x 500 Fortran order) and the common
    starting state: the rank-64 truncated SVD of snapshots 1-100 (k = 100)."""
    wl = _workloads()
    t0 = time.perf_counter()
    x, _, _, _ = wl.cfg2_stream_numpy(n=N_S, cols=COLS, rank=RANK, seed=0)
    q, r = np.linalg.qr(x[:, :WARM_COLS])
    w, s, vt = np.linalg.svd(r)
    phi = np.ascontiguousarray(q @ w[:, :RANK])
    start = dict(phi=phi, sigma=s[:RANK].copy(), v=np.ascontiguousarray(vt.T[:, :RANK]), k=WARM_COLS)
    return x, start, time.perf_counter() - t0


def host_info():
    model = platform.processor() or ""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    blas = {}
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = {"name": b.get("name"), "version": b.get("version")}
    except Exception:
        pass
    try:
        import scipy

        sv = scipy.__version__
    except Exception:
        sv = None
    return {"cpu_model": model, "cores": os.cpu_count(), "numpy": np.__version__, "scipy": sv, "blas": blas,
            "threads": os.environ.get("OPENBLAS_NUM_THREADS", "all (OpenBLAS default)")}


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and "Active" in r[4 + i]
                          and "Not" not in r[4 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "sm_mhz_min": min(sm) if sm else None, "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------------------- dist
def dist_setup(want_gpus, backend=None):
    """One process per GPU (torchrun env).  backend defaults to nccl; the CPU
    tests drive the same helpers over gloo."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist

        backend = backend or "nccl"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()


def allmax(ws, x):
    """Max over ranks (the timing rule: the slowest rank's device time)."""
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(units_per_rank_step, steps, ws, ms_max):
    """value: units processed by ALL ranks / the slowest rank's device time."""
    return units_per_rank_step * steps * ws / (ms_max / 1e3)


def replica_seed(rank):
    """Replicas only: every rank ingests the cfg2 stream of numpy seed 0 (same
    bytes as the reference arm); the extra robustness seeds are 1 and 2."""
    return 0


def config_block(ws):
    return {"workload": WORKLOAD, "n_s": N_S, "rank": RANK, "snapshots_per_step": COLS - WARM_COLS,
            "l2": "inputs larger than L2 (U >= 512 MB, X 4.2 GB); no flush",
            "parallelism": f"replicas x{ws}" if ws > 1 else "single process"}


# --------------------------------------------------------------------------- device arm
def _prof_read(lib, capi):
    pl = (capi.i64 * 16)()
    pms = (capi.dbl * 16)()
    pby = (capi.dbl * 16)()
    lib.strom_profile_read(16, pl, pms, pby)
    return list(pl), list(pms), list(pby)


SKIP_LAUNCH_MS = 0.03  # a pass that streams U at n_s = 2^20 takes > 0.1 ms; an early return < 0.02 ms


def _prof_durations(lib, capi, kind, cap=1 << 16):
    import ctypes as C

    buf = (C.c_float * cap)()
    n = C.c_int32()
    lib.strom_profile_durations(kind, cap, buf, C.byref(n))
    return [float(buf[i]) for i in range(min(cap, n.value))]


def time_ingest(start_state, cols, steps, warmup, ws=1, clocks=False):
    """Warm-up + `steps` timed ingests of `cols` from `start_state`; CUDA events
    on the launching (current) stream; returns (ms total, last state, launches,
    clock summary)."""
    import torch

    from paper_1910_01260_b200 import _capi, basis

    for _ in range(warmup):
        last = basis.ingest_simulation(start_state, cols)
    torch.cuda.synchronize()
    barrier(ws)
    torch.cuda.synchronize()
    lib = _capi.lib
    lib.strom_profile_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clk = ClockSampler(torch.cuda.current_device()) if clocks else None
    if clk:
        clk.__enter__()
    try:
        e0.record()
        for _ in range(steps):
            last = basis.ingest_simulation(start_state, cols)
        e1.record()
        torch.cuda.synchronize()
    finally:
        if clk:
            clk.__exit__(None, None, None)
    barrier(ws)
    pl, _, _ = _prof_read(lib, _capi)
    launches = int(sum(pl[k] for k in range(len(PROF_KINDS))))
    return e0.elapsed_time(e1), last, launches, (clk.summary() if clk else None)


def counts_of(state, prof_launches):
    inf = state.info()
    return {"n_dependent": int(inf.n_dependent), "n_truncated": int(inf.n_truncated),
            "compactions": int(prof_launches[PROF_KINDS.index("compact_sweep")]), "final_rank": int(inf.rank)}


def bench_isvd_device(args, ws, rank):
    import torch

    from paper_1910_01260_b200 import _capi, basis

    dev = torch.device("cuda", torch.cuda.current_device())
    xh, start, gen_s = cfg2_host()
    xd = torch.as_tensor(xh[:, WARM_COLS:], device=dev)  # X is Fortran order: columns stay contiguous
    cols = xd  # (n, 400) view, column-major
    st100 = basis.SvdState(start["phi"], start["sigma"], start["v"], start["k"], TOL, tol_sv=TOL, r_max=RANK,
                           cap_mode="truncate")
    nsnap = cols.shape[1]
    ms, last, launches, clocks = time_ingest(st100, cols, args.steps, args.warmup, ws, clocks=True)
    ms_max = allmax(ws, ms)
    value = whole_job_rate(nsnap, args.steps, ws, ms_max)
    lib = _capi.lib
    # ---- profiled repetition: per-kernel CUDA-event durations + algorithmic bytes
    lib.strom_profile_reset()
    lib.strom_profile_enable(1)
    prof_last = basis.ingest_simulation(st100, cols)
    torch.cuda.synchronize()
    lib.strom_profile_enable(0)
    pl, pms, pby = _prof_read(lib, _capi)
    kernels = {PROF_KINDS[k]: {"launches": int(pl[k]), "ms": round(pms[k], 4),
                               "gbs": (pby[k] / (pms[k] / 1e3) / 1e9) if pms[k] > 0 and pby[k] > 0 else None,
                               "bytes": pby[k] or None}
               for k in range(len(PROF_KINDS)) if pl[k]}
    # A pass launched for a snapshot that the device-side decision found dependent returns
    # at once and moves no bytes (window mode, DESIGN 3a): split the per-launch event times
    # of the byte-counting passes into the launches that streamed U and the ones that did not.
    pms = list(pms)
    for name in ("u_pass",):
        k = PROF_KINDS.index(name)
        if not pl[k] or not pby[k]:
            continue
        durs = _prof_durations(lib, _capi, k)
        live = [t for t in durs if t >= SKIP_LAUNCH_MS]
        if durs and live and len(live) < len(durs):
            kernels[name].update({"ms_all_launches": kernels[name]["ms"], "ms": round(sum(live), 4),
                                  "launches_with_work": len(live),
                                  "launches_skipped_on_device": len(durs) - len(live),
                                  "skipped_ms": round(sum(durs) - sum(live), 4),
                                  "gbs": pby[k] / (sum(live) / 1e3) / 1e9,
                                  "note": f"ms / gbs over the launches that streamed U (event time >= "
                                          f"{SKIP_LAUNCH_MS} ms); a skipped launch moves no bytes"})
            pms[k] = sum(live)
    seed0 = dict(seed="numpy 0", snapshots_per_s=value / ws, **counts_of(prof_last, pl))
    del prof_last
    info = last.info()
    return dict(value=value, ms=ms_max, nsnap=nsnap, gpu_launches=launches, clocks=clocks, kernels=kernels,
                prof=(pl, pms, pby), st100=st100, start=start, xh=xh, xd=xd, gen_s=gen_s, seed0=seed0,
                final=dict(rank=int(info.rank), n_dependent=int(info.n_dependent),
                           n_truncated=int(info.n_truncated), sigma0=float(last.sigma[0]),
                           sigma63=float(last.sigma[-1])))


def bench_isvd_seeds(args, ctx):
    """The same step on streams of torch seeds 1 and 2 (same construction,
    generated on the device), each from its own truncated SVD of snapshots 1-100."""
    import torch

    from paper_1910_01260_b200 import _capi, basis

    wl = _workloads()
    out = [ctx["seed0"]]
    dev = torch.device("cuda", torch.cuda.current_device())
    for seed in (1, 2):
        xt, _, _, _ = wl.cfg2_stream_torch(n=N_S, cols=COLS, rank=RANK, seed=seed, device=dev)
        q, r = torch.linalg.qr(xt[:WARM_COLS].T)
        w, s, vt = torch.linalg.svd(r)
        st = basis.SvdState((q @ w[:, :RANK]).contiguous(), s[:RANK], vt.T[:, :RANK].contiguous(), WARM_COLS,
                            TOL, tol_sv=TOL, r_max=RANK, cap_mode="truncate")
        del q, r, w, vt
        cols = xt[WARM_COLS:].T
        # three steps timed one by one, median: a step is ~60 ms of mostly one-CTA latency work
        # and the box's host or clock hiccups show up as single slow steps (DESIGN 3a)
        step_ms = []
        for rep in range(3):
            ms, last, _, _ = time_ingest(st, cols, 1, 2 if rep == 0 else 0)
            step_ms.append(ms)
        pl, _, _ = _prof_read(_capi.lib, _capi)
        rate = (COLS - WARM_COLS) / (statistics.median(step_ms) / 1e3)
        c = counts_of(last, pl)  # the profile counters cover the last timed step
        out.append(dict(seed=f"torch {seed}", snapshots_per_s=rate,
                        step_ms=[round(v, 2) for v in step_ms], **c))
        del xt, cols, st, last
        torch.cuda.empty_cache()
    rates = [o["snapshots_per_s"] for o in out]
    return {"per_seed": out, "median_snapshots_per_s": statistics.median(rates), "min": min(rates),
            "max": max(rates)}


def bench_isvd_e2e(args, ctx, pinned=True):
    import torch

    from paper_1910_01260_b200 import basis

    xh = ctx["xh"]
    if pinned:
        host = torch.empty((COLS - WARM_COLS, N_S), dtype=torch.float64, pin_memory=True)
        host.copy_(torch.from_numpy(xh[:, WARM_COLS:].T))
        cols_h = host.T  # (n, 400) host view, columns contiguous
    else:
        cols_h = xh[:, WARM_COLS:]  # the caller's numpy array itself (pageable)
    st100 = ctx["st100"]

    def step():
        s = basis.ingest_simulation(st100, cols_h)
        return s.sigma.cpu()  # D2H of the step result

    # at least 4 untimed steps: the first host-path calls of a process phase
    # show sporadic stalls outside the kernels
    for _ in range(max(4, args.warmup)):
        step()
    torch.cuda.synchronize()
    steps = args.steps if pinned else max(2, args.steps // 2)
    step_s = []
    with ClockSampler(torch.cuda.current_device()) as clk:
        t0 = time.perf_counter()
        for _ in range(steps):
            ts = time.perf_counter()
            sig = step()
            step_s.append(time.perf_counter() - ts)  # (sigma.cpu() has synchronised)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    nsnap = COLS - WARM_COLS
    return {"value": nsnap * steps / dt, "unit": "snapshots/s",
            "step_ms": [round(v * 1e3, 1) for v in step_s], "clocks": clk.summary(),
            "value_at_median_step": nsnap / statistics.median(step_s),
            "h2d_bytes_per_step": int(nsnap * N_S * 8), "d2h_bytes_per_step": int(sig.numel() * 8),
            "path": ("ingest_simulation(pinned host X) -> chunked H2D on a copy stream overlapped with the "
                     "updates; sigma read back") if pinned else
                    ("ingest_simulation(pageable numpy X, the reference callers' case) -> the library stages "
                     "it through pinned buffers; sigma read back")}


def cpu_baseline_isvd(ctx, budget_s=20.0):
    """Oracle port (numpy/OpenBLAS, all host threads) from the common start
    state, snapshots 101, 102, ... for about budget_s seconds."""
    from oracle import strom_oracle as so

    start, xh = ctx["start"], ctx["xh"]
    r = _oracle_updates(so, start, xh, WARM_COLS, 10 ** 6, budget_s)
    return {"value": r["rate"], "unit": "snapshots/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"oracle isvd_update on cfg2 snapshots {WARM_COLS + 1}-{WARM_COLS + r['done']} from the common "
                      f"start state ({r['done']} updates, {r['qr']} drift QRs, {r['dt']:.1f} s)",
            "rate_without_qr_updates": r["rate_noqr"], "qr_updates": r["qr"], "host": host_info()}


def _oracle_updates(so, start, xh, col0, count, budget_s=None, st=None):
    """Run `count` oracle updates from column col0 (or until budget_s); time QR
    and non-QR updates apart."""
    if st is None:
        st = so.OState(phi=start["phi"], sigma=start["sigma"], v=start["v"], k=start["k"], tol_svd=TOL,
                       tol_sv=TOL, r_max=RANK, cap_mode="truncate")
    t_qr = t_plain = 0.0
    n_qr = n_plain = 0
    t0 = time.perf_counter()
    for j in range(col0, col0 + count):
        d = so.Decision()
        ta = time.perf_counter()
        st = so.update(st, np.ascontiguousarray(xh[:, j]), d)
        tb = time.perf_counter() - ta
        if d.qr:
            t_qr += tb
            n_qr += 1
        else:
            t_plain += tb
            n_plain += 1
        if budget_s is not None and time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    done = n_qr + n_plain
    return {"st": st, "done": done, "dt": dt, "rate": done / dt if dt > 0 else 0.0, "qr": n_qr,
            "rate_noqr": n_plain / t_plain if t_plain > 0 else None, "t_qr": t_qr, "t_plain": t_plain}


def fp64_peak_tflops():
    import torch

    from paper_1910_01260_b200 import _capi

    flops = _capi.dbl()
    _capi.lib.strom_fp64_probe(200, 4, _capi.stream_ptr(), flops)  # warm
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _capi.check(_capi.lib.strom_fp64_probe(4000, 4, _capi.stream_ptr(), flops))
    e1.record()
    torch.cuda.synchronize()
    return flops.value / (e0.elapsed_time(e1) / 1e3) / 1e12


def bench_st_device(args, with_cpu):
    import torch

    from paper_1910_01260_b200 import BasisSet, LinearDynamicalSystem, TimeGrid, spacetime, spatial

    wl = _workloads()
    d = wl.cfg4_inputs()
    dev = torch.device("cuda", torch.cuda.current_device())

    def make(host):
        sys_ = LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)
        if host:
            return sys_, BasisSet(d.phi_s, d.temporal, n_mu=20), TimeGrid(d.dt)
        phi_cm = torch.as_tensor(np.asfortranarray(d.phi_s).T.copy(), device=dev).T  # column-major N x n_s
        bs = BasisSet(phi_cm, torch.as_tensor(np.stack(d.temporal), device=dev), n_mu=20)
        grid = TimeGrid(d.dt)
        sys_.device_arrays()
        grid.dt_device()
        return sys_, bs, grid

    sys_, bs, grid = make(False)

    def build():
        srom = spatial.build_spatial_rom(sys_, bs, ref_mode="zero")
        return spacetime.build_st_rom(srom, bs, grid, sys_.input_signal, True)

    for _ in range(max(args.warmup, 3)):
        rom = build()
    torch.cuda.synchronize()
    times = []
    for _ in range(max(args.steps, 5)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rom = build()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = statistics.median(times)
    from paper_1910_01260_b200 import _capi

    _capi.lib.strom_profile_reset()
    _capi.lib.strom_profile_enable(1)
    build()
    torch.cuda.synchronize()
    _capi.lib.strom_profile_enable(0)
    pl, pms, _ = _prof_read(_capi.lib, _capi)
    solve_t = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x = spacetime.solve_st_rom(rom)
        e1.record()
        torch.cuda.synchronize()
        solve_t.append(e0.elapsed_time(e1))
    # reconstruct_states on the device (spacetime.py:165-186): N x n_s x N_t
    rec_t = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        states = spacetime.reconstruct_states(bs, x)
        e1.record()
        torch.cuda.synchronize()
        rec_t.append(e0.elapsed_time(e1))
    del states
    # end to end from host data: LinearDynamicalSystem(host CSR) + BasisSet(host
    # Phi_s, Psi) -> build -> the operators read back (pipeline.run_at_param)
    e2e_t = []
    for i in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        hs, hb, hg = make(True)
        srom = spatial.build_spatial_rom(hs, hb, ref_mode="zero")
        hrom = spacetime.build_st_rom(srom, hb, hg, hs.input_signal, True)
        outs = [hrom.a_st_hat.cpu(), hrom.f_st_hat.cpu(), hrom.x0_st_hat.cpu()]
        torch.cuda.synchronize()
        if i:
            e2e_t.append((time.perf_counter() - t0) * 1e3)
        del hs, hb, hg, srom, hrom
    nnz, n, ns, nt, nsteps = d.a.nnz, d.a.shape[0], 50, 20, 500
    bytes_alg = (8 + 4) * nnz + 4 * (n + 1) + 8 * n * ns + 8 * 2 * n + 8 * ns * nsteps * nt + 8 * (ns * nt) ** 2
    flops_alg = 2 * nnz * ns + 2 * n * ns * (ns + 3) + 2 * nsteps * (ns * nt) ** 2
    h2d = (8 + 4) * nnz + 4 * (n + 1) + 8 * n * ns + 8 * 3 * n + 8 * ns * nsteps * nt + 8 * nsteps
    out = {"metric": "ST-ROM operator build ms", "value": ms, "unit": "ms", "higher_is_better": False,
           "solve_ms": statistics.median(solve_t),
           "reconstruct_states_ms": statistics.median(rec_t),
           "workload": "cfg4: 3D 7-point adv-diff 100^3 (nnz 6.94M, int32 CSR), n_s=50, n_t=20, N_t=500, "
                       "ref_mode=zero, constant input",
           "algorithmic_bytes": bytes_alg, "algorithmic_flops": flops_alg,
           "kernels_ms": {"spatial_spmm_gram": round(pms[7], 4), "st_temporal_gram": round(pms[8], 4)},
           "e2e": {"value": statistics.median(e2e_t), "unit": "ms", "h2d_bytes_per_step": int(h2d),
                   "d2h_bytes_per_step": int(8 * ((ns * nt) ** 2 + 2 * ns * nt)),
                   "path": "LinearDynamicalSystem(host CSR) + BasisSet(host Phi_s, Psi) -> build_spatial_rom -> "
                           "build_st_rom -> A_st, f_st, x0_st read back; CSR->tiled-ELL conversion included"}}
    if with_cpu:
        from oracle import strom_oracle as so

        ct = []
        for _ in range(3):
            t0 = time.perf_counter()
            o = so.spatial_rom(d.a, d.b, d.c, d.x0, d.phi_s, "zero")
            so.st_matrix(o.a_hat, d.temporal, d.dt)
            so.st_input(o.b_hat, d.temporal, d.dt, d.inputs, True)
            so.st_init(o.x0_hat, d.temporal)
            ct.append(time.perf_counter() - t0)
        out["cpu_baseline"] = {"value": statistics.median(ct) * 1e3, "unit": "ms", "cores": os.cpu_count(),
                               "kind": "port",
                               "sample": "oracle build_spatial_rom + build_st_matrix/input/init at full cfg4 size, "
                                         "median of 3 (SciPy CSR x dense is single-threaded)"}
    del x
    return out


def bench_cfg1(args, with_cpu):
    """BASELINE configs[0] whole pipeline: 4 training marches -> iSVD -> temporal
    bases -> spatial ROM at the test nu -> ST build -> solve -> lift (the
    reference's train + run_at_param, pipeline.py:76-124, 240-256)."""
    import torch

    from paper_1910_01260_b200 import (LinearDynamicalSystem, TimeGrid, basis, fom_march, spacetime,
                                       spatial)

    wl = _workloads()

    def lds(d):
        return LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)

    grid = TimeGrid(wl.cfg1_dt())
    train = [lds(wl.cfg1_system(nu)) for nu in wl.CFG1_TRAIN_NU]
    test = lds(wl.cfg1_system(wl.CFG1_TEST_NU))
    for s_ in train + [test]:
        s_.device_arrays()
    grid.dt_device()

    def run():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record()
        mats = [fom_march(s_, grid).states for s_ in train]
        ev[1].record()
        st = basis.isvd_init(mats[0][:, 0], wl.CFG1_TOL, tol_sv=wl.CFG1_TOL)
        st = basis.ingest_simulation(st, mats[0][:, 1:])
        for m in mats[1:]:
            st = basis.ingest_simulation(st, m)
        ev[2].record()
        bs = basis.build_basis_set(st, wl.CFG1_NS, wl.CFG1_NTMODES, wl.CFG1_NT, len(wl.CFG1_TRAIN_NU))
        ev[3].record()
        srom = spatial.build_spatial_rom(test, bs, ref_mode="zero")
        rom = spacetime.build_st_rom(srom, bs, grid, test.input_signal, True)
        ev[4].record()
        x_st = spacetime.solve_st_rom(rom)
        states = spacetime.reconstruct_states(bs, x_st)
        ev[5].record()
        torch.cuda.synchronize()
        return [ev[i].elapsed_time(ev[i + 1]) for i in range(5)], ev[0].elapsed_time(ev[5]), st

    run()
    runs = [run() for _ in range(5)]
    names = ["fom_4x100_steps", "isvd_400_snapshots", "temporal_bases", "st_operator_build", "st_solve_and_lift"]
    stage = {names[i]: statistics.median(r[0][i] for r in runs) for i in range(5)}
    out = {"metric": "cfg1 whole pipeline ms", "value": statistics.median(r[1] for r in runs), "unit": "ms",
           "higher_is_better": False,
           "workload": "cfg1: 1D periodic advection-diffusion, N=1024, 4 training nu x 100 backward-Euler steps, "
                       "tol 1e-8, n_s=10 x n_t=4 modes, test nu=0.025; median of 5",
           "stages_ms": stage, "isvd_us_per_snapshot": stage["isvd_400_snapshots"] * 1e3 / 400,
           "rank": runs[-1][2].rank}
    if with_cpu:
        from oracle import strom_oracle as so

        t0 = time.perf_counter()
        dt = grid.dt
        mats = [so.fom_march(d.a, d.b, d.x0, dt, d.inputs) for d in map(wl.cfg1_system, wl.CFG1_TRAIN_NU)]
        ref = so.stream(np.hstack(mats), wl.CFG1_TOL, tol_sv=wl.CFG1_TOL)
        phi_s, temporal, _ = so.basis_set(ref, wl.CFG1_NS, wl.CFG1_NTMODES, wl.CFG1_NT, 4)
        d = wl.cfg1_system(wl.CFG1_TEST_NU)
        o = so.spatial_rom(d.a, d.b, d.c, d.x0, phi_s, "zero")
        a_st = so.st_matrix(o.a_hat, temporal, dt)
        f_st = so.st_input(o.b_hat, temporal, dt, d.inputs, True)
        i_st = so.st_init(o.x0_hat, temporal)
        x_ref = so.st_solve(a_st, f_st, i_st)
        so.st_reconstruct(phi_s, temporal, x_ref)
        out["cpu_baseline"] = {"value": (time.perf_counter() - t0) * 1e3, "unit": "ms", "cores": os.cpu_count(),
                               "kind": "port", "sample": "the whole cfg1 pipeline through the oracle, one run"}
    return out


def bench_cfg3(args):
    """BASELINE configs[2] transport proxy: device FOM march (64^3 x 4 dofs, 4 x 100
    steps) feeding the device iSVD, then temporal bases (tools/cfg3_transport.py)."""
    import torch

    from paper_1910_01260_b200 import LinearDynamicalSystem, TimeGrid, basis, fom_march

    wl = _workloads()
    t0 = time.time()
    a = wl.cfg3_operator()
    t_op = time.time() - t0
    grid = TimeGrid(np.full(wl.CFG3_NT, wl.CFG3_DT))
    st = None
    fom_ms, ingest_ms, iters = [], [], []
    for amp in wl.CFG3_AMPLITUDES:
        d = wl.cfg3_system(amp, a=a)
        sys_ = LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)
        sys_.device_arrays()
        # The GPU idles while the host assembles each sample's system and drops its clocks
        # (clocks_throttle_reasons gpu_idle, 120-900 MHz seen); one-CTA latency phases then run
        # several times slower for a while.  So: one untimed repetition to bring the clocks
        # back, then the march once and the (functional: the source state is immutable)
        # ingest three times, median.
        fom_march(sys_, grid)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        res = fom_march(sys_, grid)
        e[1].record()
        reps = []
        for rep in range(4):
            ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ea.record()
            if st is None:
                nxt = basis.ingest_simulation(basis.isvd_init(res.states[:, 0], wl.CFG3_TOL, tol_sv=wl.CFG3_TOL),
                                              res.states[:, 1:])
            else:
                nxt = basis.ingest_simulation(st, res.states)
            eb.record()
            torch.cuda.synchronize()
            if rep:
                reps.append(ea.elapsed_time(eb))
        st = nxt
        fom_ms.append(e[0].elapsed_time(e[1]))
        ingest_ms.append(float(np.median(reps)))
        iters += res.iterations
        del res
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    bs = basis.build_basis_set(st, min(10, st.rank), 2, wl.CFG3_NT, len(wl.CFG3_AMPLITUDES))
    e1.record()
    torch.cuda.synchronize()
    nsnap = wl.CFG3_NT * len(wl.CFG3_AMPLITUDES)
    return {"workload": "cfg3 transport proxy: 64^3 cells x 4 directions (2^20 dofs), sigma_t 1, sigma_s 0.5, "
                        "backward Euler dt 0.01, 100 steps x amplitudes {0.5,1,1.5,2}, iSVD tol 1e-8, n_t=2",
            "fom_ms_per_step": sum(fom_ms) / nsnap, "bicgstab_iterations_mean": float(np.mean(iters)),
            "isvd_snapshots_per_s": nsnap / (sum(ingest_ms) / 1e3), "rank": st.rank,
            "temporal_bases_ms": e0.elapsed_time(e1), "device_total_ms": sum(fom_ms) + sum(ingest_ms) +
            e0.elapsed_time(e1), "operator_assembly_s_host": t_op,
            "ingest_ms_per_sample": [round(v, 3) for v in ingest_ms],
            "timing": "per sample: one untimed march (GPU clocks back up after the host-side assembly), the march "
                      "timed once, the ingest median of 3 after one untimed repetition",
            "note": "the reference cannot produce these snapshots (SuperLU fill-in; SURVEY 8(d))"}


def bench_cfg5(args, ncols=400, timed_from=100):
    """BASELINE configs[4] capacity run, bounded: n_s = 2^26, rank-100 stream generated
    on the device in batches of 8 outside the timed region; updates timed_from..ncols-1
    timed (rank pinned at 100 by then).  tools/cfg5_capacity.py runs all 1000."""
    import math

    import torch

    from paper_1910_01260_b200 import basis

    wl = _workloads()
    n, B = 1 << 26, 8
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = wl.HadamardStream(n, 1000, 100, decades_per=12.0, seed=0)
    buf = torch.empty((B, n), dtype=torch.float64, device=dev)
    st = basis.isvd_init(stream.batch(0, 1, out=buf[:1])[:, 0], TOL, tol_sv=TOL, r_max=100, cap_mode="truncate")
    t0, timed_ms, timed_n = 1, 0.0, 0
    call_ms = []
    clk = ClockSampler(torch.cuda.current_device())
    clk.__enter__()
    try:
        while t0 < ncols:
            nb = 1 << int(math.floor(math.log2(min(B, ncols - t0))))
            xb = stream.batch(t0, nb, out=buf[:nb])
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            st = basis.ingest_simulation(st, xb)
            e1.record()
            torch.cuda.synchronize()
            if t0 >= timed_from:
                timed_ms += e0.elapsed_time(e1)
                timed_n += nb
                if nb == B:
                    call_ms.append(e0.elapsed_time(e1))
            t0 += nb
    finally:
        clk.__exit__(None, None, None)
    # singular values of this prefix of the stream: X[:, :ncols] = Q diag(sigma) W[:ncols]^T + E
    # (the W rows of a prefix are not orthonormal, so they differ from sigma)
    known = torch.linalg.svdvals(stream.w[:ncols] * stream.sigma)
    sig = st.sigma
    rel = ((sig[:16] - known[:16]).abs() / known[:16]).cpu()
    c_avg = None
    out = {"workload": f"cfg5 capacity: n_s=2^26 fp64, rank-100 stream (sigma_i=10^(-i/12), noise 1e-12), "
                       f"r_max=100 truncate, tol 1e-9; snapshots {timed_from}-{ncols - 1} timed of a {ncols}-snapshot "
                       "prefix of the 1000-snapshot stream",
           "snapshots_per_s": timed_n / (timed_ms / 1e3), "ms_per_update": timed_ms / timed_n,
           "rank": st.rank, "sigma_rel_err_max_i_lt_16_vs_prefix_svd": float(rel.max()),
           "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9,
           "floor_frac_of_hbm": None,
           "ms_per_8_column_call": {"median": statistics.median(call_ms) if call_ms else None,
                                    "max": max(call_ms) if call_ms else None,
                                    "note": "calls with a compaction are the slow ones"},
           "clocks": clk.summary()}
    bw, _ = peaks()
    out["floor_frac_of_hbm"] = out["snapshots_per_s"] * 8.0 * n * 101 / (bw * 1e9)
    del st, buf, sig, c_avg
    return out


def _guarded(name, fn, *a, **kw):
    """Secondary measurements must not cost the primary line: a failure is
    reported in its key (and on stderr) instead of aborting the run."""
    try:
        return fn(*a, **kw)
    except Exception as e:  # noqa: BLE001
        import traceback

        traceback.print_exc()
        return {"error": f"{name}: {type(e).__name__}: {e}"}


def run_device(args):
    import torch

    ws, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    bw, bw_src = peaks()
    ctx = bench_isvd_device(args, ws, rank)
    kern = ctx["kernels"]
    # dominant HBM kernel of the step (by event time) and its live roofline.  Only
    # kernels that count algorithmic bytes qualify: the core step on the second
    # stream starts early and spins on a device counter, so its event time
    # includes waiting and says nothing about its own cost.
    pl, pms, pby = ctx["prof"]
    dom = max(range(len(PROF_KINDS)), key=lambda k: pms[k] if pby[k] > 0 else -1.0)
    achieved = pby[dom] / (pms[dom] / 1e3) / 1e9 if pms[dom] > 0 else 0.0
    traffic = None
    tpath = os.path.join(HERE, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(PROF_KINDS[dom])
        except Exception:
            traffic = None
    nsnap = ctx["nsnap"]
    per_rank_rate = ctx["value"] / ws
    dev_bytes_step = float(sum(b for b in pby if b))           # every HBM kernel's algorithmic bytes, one step
    floor_bytes = 8.0 * N_S * (RANK + 1)                       # read Phi once + x, any algorithm
    b_ref = 8.0 * N_S * (3 * RANK + 2)                         # the reference's direct form
    step_ms = ctx["ms"] / args.steps
    line = {
        "metric": METRIC,
        "value": ctx["value"],
        "unit": "snapshots/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE config 2 construction, numpy default_rng(0), same bytes as the reference arm)",
        "config": config_block(ws),
        "roofline": {"bound": "hbm", "kernel": PROF_KINDS[dom], "achieved": achieved, "peak": bw,
                     "peak_source": bw_src, "unit": "GB/s", "frac": achieved / bw, "traffic": traffic,
                     "step_frac": dev_bytes_step / (step_ms / 1e3) / 1e9 / bw,
                     "step_bytes_per_snapshot": dev_bytes_step / nsnap,
                     "floor_frac": per_rank_rate * floor_bytes / (bw * 1e9),
                     "floor_bytes_per_snapshot": floor_bytes,
                     "note": "frac: the dominant kernel's algorithmic bytes / its event time over the launches "
                             "that did work (kernels.*.launches_skipped_on_device returned at once); step_frac: all of "
                             "the step's device HBM bytes / step time; floor_frac: snapshots/s x 8 n (k+1) (read Phi "
                             "and x once: the any-algorithm floor of SURVEY 8(d)) / peak"},
        "north_star": {"target": ">= 0.70 of the HBM roofline at n_s=2^20, k=64",
                       "frac_of_floor": per_rank_rate * floor_bytes / (bw * 1e9),
                       "reference_traffic_speed_equiv": per_rank_rate * b_ref / (bw * 1e9),
                       "note": "reference_traffic_speed_equiv = snapshots/s x B_ref / peak with B_ref = 8 n (3k+2), "
                               "the bytes the REFERENCE's direct form moves; not a hardware fraction (the device "
                               "moves step_bytes_per_snapshot)"},
        "kernels": kern,
        "gpu_launches": ctx["gpu_launches"],
        "clocks": ctx["clocks"],
        "final_state": ctx["final"],
        "input_generation_s_untimed": ctx["gen_s"],
    }
    if rank == 0 and not args.no_e2e:
        line["e2e"] = bench_isvd_e2e(args, ctx, pinned=True)
        line["e2e_pageable"] = bench_isvd_e2e(args, ctx, pinned=False)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_isvd(ctx)
    seed0 = ctx["seed0"]
    ctx.pop("xd", None)
    if rank == 0 and ws == 1 and not args.no_seeds:
        line["seeds"] = _guarded("seeds", bench_isvd_seeds, args, ctx)
    else:
        line["seeds"] = {"per_seed": [seed0]}
    del ctx
    torch.cuda.empty_cache()
    if rank == 0 and not args.skip_st:
        st = bench_st_device(args, with_cpu=(ws == 1 and not args.no_cpu_baseline))
        peak64 = fp64_peak_tflops()
        t = st["value"] / 1e3
        floor_t = max(st["algorithmic_bytes"] / (bw * 1e9), st["algorithmic_flops"] / (peak64 * 1e12))
        st["roofline"] = {"bound": "fp64 tensor + hbm (combined)", "achieved_floor_ms": floor_t * 1e3,
                          "frac": floor_t / t, "fp64_peak_tflops_measured": peak64,
                          "hbm_peak_gbs": bw, "note": "max(bytes/BW, flops/P_fp64) / t (SURVEY 8(d))"}
        line["st_build"] = st
        torch.cuda.empty_cache()
    if rank == 0 and not args.skip_extra:
        line["cfg1"] = _guarded("cfg1", bench_cfg1, args, with_cpu=(ws == 1 and not args.no_cpu_baseline))
        torch.cuda.empty_cache()
        line["cfg3"] = _guarded("cfg3", bench_cfg3, args)
        torch.cuda.empty_cache()
        if not args.skip_cfg5:
            line["cfg5"] = _guarded("cfg5", bench_cfg5, args)
            torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- row-sharded stream
def run_sharded(args):
    """The cfg2 stream row-sharded over the ranks of one NVSwitch domain:
    every rank owns n / G rows of U and of each snapshot, sigma / V / decisions are replicated,
    the per-rank partial sums cross the GPUs in one small kernel over peer-memory mailboxes.
    Strong scaling: total work fixed.  At G = 1 the exchange degenerates to a copy through the
    mailbox: the line then measures the protocol's overhead against the unsharded run."""
    import torch

    ws, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    from paper_1910_01260_b200 import basis
    from paper_1910_01260_b200.sharded import ShardGroup

    dev = torch.device("cuda", local)
    xh, start, gen_s = cfg2_host()
    group = ShardGroup.connect(N_S)
    r0, nl = group.row0, group.n_local
    xd = torch.as_tensor(np.ascontiguousarray(xh[r0:r0 + nl, WARM_COLS:].T), device=dev).T  # n_local x 400, col-major
    with group:
        st100 = basis.SvdState(np.ascontiguousarray(start["phi"][r0:r0 + nl]), start["sigma"], start["v"], start["k"],
                               TOL, tol_sv=TOL, r_max=RANK, cap_mode="truncate")
    ms, last, launches, clocks = time_ingest(st100, xd, args.steps, args.warmup, ws, clocks=(rank == 0))
    ms_max = allmax(ws, ms)
    nsnap = COLS - WARM_COLS
    info = last.info()
    nex, err = group.status()
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "mode": "row-sharded (one stream over all ranks)", "value": nsnap * args.steps /
            (ms_max / 1e3), "unit": "snapshots/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (BASELINE config 2 construction, numpy default_rng(0))",
            "config": dict(config_block(1), parallelism=f"row-sharded x{ws}", rows_per_rank=nl),
            "gpu_launches": launches, "clocks": clocks, "exchanges": nex, "exchange_errors": err,
            "final_state": dict(rank=int(info.rank), n_dependent=int(info.n_dependent),
                                n_truncated=int(info.n_truncated), sigma0=float(last.sigma[0]))}), flush=True)
    barrier(ws)


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The reference's algorithm (oracle port, bit-identical to strom.basis in this
    image) on the device arm's workload: same bytes, same start state, each step
    two consecutive updates from snapshot 101.  Rank 0 only under torchrun."""
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import strom_oracle as so

    per_step = 2
    xh, start, gen_s = cfg2_host()
    col = WARM_COLS
    st = None
    for _ in range(args.warmup):
        r = _oracle_updates(so, start, xh, col, per_step, st=st)
        st, col = r["st"], col + per_step
    first_timed = col + 1
    t_qr = t_plain = 0.0
    n_qr = n_plain = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        r = _oracle_updates(so, start, xh, col, per_step, st=st)
        st, col = r["st"], col + per_step
        t_qr += r["t_qr"]
        t_plain += r["t_plain"]
        n_qr += r["qr"]
        n_plain += r["done"] - r["qr"]
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "snapshots/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config 2 construction, numpy default_rng(0), same bytes as the device arm)",
            "config": config_block(ws),
            "cpu_baseline": {"value": value, "unit": "snapshots/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": f"{per_step} consecutive isvd_update calls per step; snapshots "
                                       f"{WARM_COLS + 1}-{first_timed - 1} warm-up, {first_timed}-{col} timed "
                                       f"({n_qr} drift QRs); input generation {gen_s:.1f} s untimed",
                             "rate_without_qr_updates": (n_plain / t_plain) if t_plain > 0 else None,
                             "rate_qr_updates": (n_qr / t_qr) if t_qr > 0 else None,
                             "qr_updates": n_qr, "host": host_info()},
            "e2e": {"value": value, "unit": "snapshots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--skip-st", action="store_true")
    ap.add_argument("--skip-extra", action="store_true", help="no cfg1 / cfg3 / cfg5 keys")
    ap.add_argument("--skip-cfg5", action="store_true")
    ap.add_argument("--no-seeds", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="one cfg2 stream ROW-SHARDED over the ranks (sharded.ShardGroup, strong scaling) "
                         "instead of one replica per rank; prints its own JSON line")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.shard:
        run_sharded(args)
    else:
        run_device(args)


if __name__ == "__main__":
    main()
