#!/usr/bin/env python
"""Benchmark of the B200 hot path on the BASELINE.json workloads.

Metric (BASELINE.json): "iSVD snapshots/s at n_s=1M fp64 (% HBM roofline);
ST-ROM operator build ms".

* Primary line (``value``): device iSVD ingestion on config 2 -- n_s = 2^20,
  500-snapshot low-rank-plus-noise stream, tol_svd = tol_sv = 1e-9,
  r_max = 64 (truncate).  One step = ``ingest_simulation`` of the steady-state
  snapshots 101-500 (rank pinned at 64) starting from the state after 100
  snapshots; inputs are HBM-resident; U (>= 512 MB) and X (4.2 GB) exceed L2,
  so no flush is needed.  value = snapshots/s over all ranks.
* ``e2e``: the same step through the public API from pinned HOST memory
  (chunked H2D overlapped with the updates inside the C ABI) plus the D2H
  read of sigma.
* ``st_build``: config 4 operator build {A_hat, B_hat, x0_hat, A_st, f_st,
  x0_st} from (A, Phi_s, Psi, dt, B, x0), N = 10^6, n_s = 50, n_t = 20,
  N_t = 500, ms per build; the dense solve is reported separately.
* ``cpu_baseline``: the CPU oracle port (numpy/OpenBLAS, all host cores) on a
  bounded sample of the same workloads, rank 0, N = 1.

``--impl reference`` times the oracle port alone (the reference is pure
Python/NumPy) and prints the same line with impl=reference.
Multi-GPU (torchrun): independent replicas, one stream per rank.
"""

from __future__ import annotations

import argparse
import json
import os
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
PROF_KINDS = ["fused_pass", "reorth_pass", "decide", "core_step", "v_update", "compact_prep", "compact_sweep",
              "spatial", "st_gemm", "st_small", "lu", "temporal", "other"]


def peaks():
    path = os.path.join(HERE, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


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
                "reasons": reasons, "samples": len(self.rows)}


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
    """Replicas only: rank r ingests its own independent cfg2 stream (seed r)."""
    return rank


# --------------------------------------------------------------------------- device arm
def bench_isvd_device(args, ws, rank):
    import torch

    from paper_1910_01260_b200 import _capi, basis, workloads as wl

    dev = torch.device("cuda", torch.cuda.current_device())
    xt, _, _, _ = wl.cfg2_stream_torch(n=N_S, cols=COLS, rank=RANK, seed=replica_seed(rank), device=dev)
    torch.cuda.synchronize()
    st0 = basis.isvd_init(xt[0], TOL, tol_sv=TOL, r_max=RANK, cap_mode="truncate")
    st100 = basis.ingest_simulation(st0, xt[1:WARM_COLS].T)
    cols = xt[WARM_COLS:].T  # (n, 400) view, columns contiguous
    nsnap = cols.shape[1]

    def step():
        return basis.ingest_simulation(st100, cols)

    for _ in range(args.warmup):
        last = step()
    torch.cuda.synchronize()
    last_rank = last.rank
    barrier(ws)
    torch.cuda.synchronize()
    lib = _capi.lib
    lib.strom_profile_reset()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        e0.record()
        for _ in range(args.steps):
            last = step()
        e1.record()
        torch.cuda.synchronize()
    barrier(ws)
    ms = e0.elapsed_time(e1)
    launches = (_capi.i64 * 16)()
    lib.strom_profile_read(16, launches, None, None)
    gpu_launches = int(sum(launches[k] for k in range(len(PROF_KINDS))))
    ms_max = allmax(ws, ms)
    value = whole_job_rate(nsnap, args.steps, ws, ms_max)
    # ---- profiled repetition: per-kernel CUDA-event durations + algorithmic bytes
    lib.strom_profile_reset()
    lib.strom_profile_enable(1)
    prof_last = step()
    torch.cuda.synchronize()
    lib.strom_profile_enable(0)
    pl = (_capi.i64 * 16)()
    pms = (_capi.dbl * 16)()
    pby = (_capi.dbl * 16)()
    lib.strom_profile_read(16, pl, pms, pby)
    kernels = {PROF_KINDS[k]: {"launches": int(pl[k]), "ms": round(pms[k], 4),
                               "gbs": (pby[k] / (pms[k] / 1e3) / 1e9) if pms[k] > 0 and pby[k] > 0 else None}
               for k in range(len(PROF_KINDS)) if pl[k]}
    del prof_last
    info = last.info()
    return dict(value=value, ms=ms_max, nsnap=nsnap, gpu_launches=gpu_launches, clocks=clk.summary(),
                kernels=kernels, prof=(list(pl), list(pms), list(pby)), st100=st100, xt=xt,
                final=dict(rank=last_rank, n_dependent=info.n_dependent, n_truncated=info.n_truncated,
                           sigma0=float(last.sigma[0]), sigma63=float(last.sigma[-1])))


def bench_isvd_e2e(args, ctx):
    import torch

    from paper_1910_01260_b200 import basis

    xt = ctx["xt"]
    host = torch.empty((COLS - WARM_COLS, N_S), dtype=torch.float64, pin_memory=True)
    host.copy_(xt[WARM_COLS:])
    cols_h = host.T  # (n, 400) host view, columns contiguous
    st100 = ctx["st100"]

    def step():
        s = basis.ingest_simulation(st100, cols_h)
        return s.sigma.cpu()  # D2H of the step result

    # at least 4 untimed steps: the first 3 host-path calls after the device
    # timing show sporadic stalls of up to ~1 s outside the kernels (between
    # launches; tools/e2e_probe.py), never a later one
    for _ in range(max(4, args.warmup)):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        sig = step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    nsnap = COLS - WARM_COLS
    return {"value": nsnap * args.steps / dt, "unit": "snapshots/s",
            "h2d_bytes_per_step": int(nsnap * N_S * 8), "d2h_bytes_per_step": int(sig.numel() * 8),
            "path": "ingest_simulation(host pinned X) -> chunked H2D on a copy stream overlapped with updates; "
                    "sigma read back"}


def cpu_baseline_isvd(ctx, budget_s=20.0, max_updates=8):
    """Oracle port (numpy/OpenBLAS, all host threads) from the device state after 100 snapshots."""
    import torch

    from oracle import strom_oracle as so

    st = ctx["st100"]
    phi = st.phi.cpu().numpy()
    ref = so.OState(phi=np.ascontiguousarray(phi), sigma=st.sigma.cpu().numpy(), v=st.v.cpu().numpy(), k=st.k,
                    tol_svd=TOL, tol_sv=TOL, r_max=RANK, cap_mode="truncate")
    cols = ctx["xt"][WARM_COLS:WARM_COLS + max_updates].cpu().numpy()
    t0 = time.perf_counter()
    done, nqr = 0, 0
    for j in range(cols.shape[0]):
        d = so.Decision()
        ref = so.update(ref, cols[j], d)
        nqr += d.qr
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": "snapshots/s", "cores": os.cpu_count(), "kind": "port",
            "sample": f"oracle isvd_update on cfg2 snapshots 101-{100 + done} from the device state after 100 "
                      f"({done} updates, {nqr} drift QRs, {dt:.1f} s)"}


def fp64_peak_tflops():
    import torch

    from paper_1910_01260_b200 import _capi

    flops = _capi.dbl()
    s = torch.cuda.current_stream()
    _capi.lib.strom_fp64_probe(200, 4, _capi.stream_ptr(), flops)  # warm
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _capi.check(_capi.lib.strom_fp64_probe(4000, 4, _capi.stream_ptr(), flops))
    e1.record()
    torch.cuda.synchronize()
    return flops.value / (e0.elapsed_time(e1) / 1e3) / 1e12


def bench_st_device(args, with_cpu):
    import torch

    from paper_1910_01260_b200 import (BasisSet, LinearDynamicalSystem, TimeGrid, spacetime, spatial,
                                       workloads as wl)

    d = wl.cfg4_inputs()
    sys_ = LinearDynamicalSystem(a=d.a, b=d.b, c=d.c, x0=d.x0, input_signal=d.inputs, constant_input=True)
    dev = torch.device("cuda", torch.cuda.current_device())
    phi_cm = torch.as_tensor(np.asfortranarray(d.phi_s).T.copy(), device=dev).T  # column-major N x n_s
    bs = BasisSet(phi_cm, torch.as_tensor(np.stack(d.temporal), device=dev), n_mu=20)
    grid = TimeGrid(d.dt)
    sys_.device_arrays()
    grid.dt_device()

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
    # kernel split of one build
    from paper_1910_01260_b200 import _capi

    _capi.lib.strom_profile_reset()
    _capi.lib.strom_profile_enable(1)
    build()
    torch.cuda.synchronize()
    _capi.lib.strom_profile_enable(0)
    pl, pms = (_capi.i64 * 16)(), (_capi.dbl * 16)()
    _capi.lib.strom_profile_read(16, pl, pms, None)
    solve_t = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        x = spacetime.solve_st_rom(rom)
        e1.record()
        torch.cuda.synchronize()
        solve_t.append(e0.elapsed_time(e1))
    nnz, n, ns, nt, nsteps = d.a.nnz, d.a.shape[0], 50, 20, 500
    bytes_alg = (8 + 4) * nnz + 4 * (n + 1) + 8 * n * ns + 8 * 2 * n + 8 * ns * nsteps * nt + 8 * (ns * nt) ** 2
    flops_alg = 2 * nnz * ns + 2 * n * ns * (ns + 3) + 2 * nsteps * (ns * nt) ** 2
    out = {"metric": "ST-ROM operator build ms", "value": ms, "unit": "ms", "higher_is_better": False,
           "solve_ms": statistics.median(solve_t),
           "workload": "cfg4: 3D 7-point adv-diff 100^3 (nnz 6.94M, int32 CSR), n_s=50, n_t=20, N_t=500, "
                       "ref_mode=zero, constant input",
           "algorithmic_bytes": bytes_alg, "algorithmic_flops": flops_alg,
           "kernels_ms": {"spatial_spmm_gram": round(pms[7], 4), "st_temporal_gram": round(pms[8], 4)}}
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
    b_ref = 8.0 * N_S * (3 * RANK + 2)  # bytes/snapshot of the reference's direct form
    line = {
        "metric": METRIC,
        "value": ctx["value"],
        "unit": "snapshots/s",
        "n_gpus": ws,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ctx["ms"] / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE config 2 construction, torch RNG on device, seed = rank)",
        "config": {"workload": "cfg2: n_s=2^20 fp64, 500-snapshot stream X=Q diag(10^(-i/8)) W^T + 1e-12 N(0,1); "
                               "tol_svd=tol_sv=1e-9, r_max=64 truncate; step = ingest snapshots 101-500",
                   "snapshots_per_step": ctx["nsnap"], "n_s": N_S, "rank": RANK,
                   "l2": "inputs larger than L2 (U >= 512 MB, X 4.2 GB); no flush",
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
        "roofline": {"bound": "hbm", "kernel": PROF_KINDS[dom], "achieved": achieved, "peak": bw,
                     "peak_source": bw_src, "unit": "GB/s", "frac": achieved / bw, "traffic": traffic},
        "north_star": {"B_ref_bytes_per_snapshot": b_ref,
                       "frac_of_measured_hbm": ctx["value"] / ws * b_ref / (bw * 1e9),
                       "frac_of_8TBs": ctx["value"] / ws * b_ref / 8.0e12,
                       "note": "SURVEY 8(d): snapshots/s x 8 n_s (3k+2) / BW; the device moves fewer bytes than "
                               "the reference's direct form (append-only U, small-space W)"},
        "kernels": kern,
        "gpu_launches": ctx["gpu_launches"],
        "clocks": ctx["clocks"],
        "final_state": ctx["final"],
    }
    if rank == 0 and not args.no_e2e:
        line["e2e"] = bench_isvd_e2e(args, ctx)
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_isvd(ctx)
    if rank == 0 and not args.skip_st:
        del ctx
        torch.cuda.empty_cache()
        st = bench_st_device(args, with_cpu=(ws == 1 and not args.no_cpu_baseline))
        peak64 = fp64_peak_tflops()
        t = st["value"] / 1e3
        floor_t = max(st["algorithmic_bytes"] / (bw * 1e9), st["algorithmic_flops"] / (peak64 * 1e12))
        st["roofline"] = {"bound": "fp64 tensor + hbm (combined)", "achieved_floor_ms": floor_t * 1e3,
                          "frac": floor_t / t, "fp64_peak_tflops_measured": peak64,
                          "hbm_peak_gbs": bw, "note": "max(bytes/BW, flops/P_fp64) / t (SURVEY 8(d))"}
        line["st_build"] = st
    if rank == 0:
        print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import strom_oracle as so
    from paper_1910_01260_b200 import workloads as wl

    per_step = 2
    t_gen = time.perf_counter()
    x, _, _, _ = wl.cfg2_stream_numpy(n=N_S, cols=WARM_COLS + per_step * (args.steps + args.warmup), rank=RANK)
    # state after 100 snapshots: exact truncated SVD of X[:, :100] (the steady-state starting point)
    q, r = np.linalg.qr(x[:, :WARM_COLS])
    w, s, vt = np.linalg.svd(r)
    st = so.OState(phi=np.ascontiguousarray(q @ w[:, :RANK]), sigma=s[:RANK], v=vt.T[:, :RANK].copy(),
                   k=WARM_COLS, tol_svd=TOL, tol_sv=TOL, r_max=RANK, cap_mode="truncate")
    gen_s = time.perf_counter() - t_gen
    col = WARM_COLS
    for _ in range(args.warmup):
        for _ in range(per_step):
            st = so.update(st, x[:, col]); col += 1
    t0 = time.perf_counter()
    nqr = 0
    for _ in range(args.steps):
        for _ in range(per_step):
            d = so.Decision()
            st = so.update(st, x[:, col], d); col += 1
            nqr += d.qr
    dt = time.perf_counter() - t0
    value = per_step * args.steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "snapshots/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config 2 construction, numpy seed 0)",
            "config": {"workload": "cfg2: n_s=2^20 fp64, tol 1e-9, r_max=64 truncate; step = 2 isvd_update calls "
                                   "on snapshots > 100 from the rank-64 SVD of the first 100",
                       "snapshots_per_step": per_step},
            "cpu_baseline": {"value": value, "unit": "snapshots/s", "cores": os.cpu_count(), "kind": "port",
                             "sample": f"{per_step * args.steps} timed oracle isvd_update calls ({nqr} drift QRs); "
                                       f"input generation {gen_s:.1f} s untimed"},
            "e2e": {"value": value, "unit": "snapshots/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--skip-st", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_device(args)


if __name__ == "__main__":
    main()
