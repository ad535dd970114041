import math, sys, time
sys.path.insert(0, '.')
import torch
from paper_1910_01260_b200 import _capi, basis, workloads as wl
KINDS = ['u_pass', 'reorth', 'decide', 'core_step', 'v_update', 'compact_prep', 'compact_sweep', 'spatial', 'st', 'lu', 'window_pass', 'other']
lib = _capi.lib
lib.strom_profile_enable(1)
n, B = 1 << 26, 8
dev = torch.device('cuda')
stream = wl.HadamardStream(n, 1000, 100, decades_per=12.0, seed=0)
buf = torch.empty((B, n), dtype=torch.float64, device=dev)
st = basis.isvd_init(stream.batch(0, 1, out=buf[:1])[:, 0], 1e-9, tol_sv=1e-9, r_max=100, cap_mode='truncate')
t0 = 1
rows = []
while t0 < 280:
    nb = 1 << int(math.floor(math.log2(min(B, 280 - t0))))
    xb = stream.batch(t0, nb, out=buf[:nb])
    torch.cuda.synchronize()
    lib.strom_profile_reset()
    w0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    st = basis.ingest_simulation(st, xb)
    e1.record()
    torch.cuda.synchronize()
    pl = (_capi.i64 * 16)(); pms = (_capi.dbl * 16)(); pby = (_capi.dbl * 16)()
    lib.strom_profile_read(16, pl, pms, pby)
    kinds = ', '.join(f'{KINDS[k]} {pms[k]:.0f}' for k in range(len(KINDS)) if pms[k] >= 5.0 and KINDS[k] != 'core_step')
    rows.append((t0, nb, e0.elapsed_time(e1), (time.perf_counter() - w0) * 1e3, kinds))
    t0 += nb
for r in rows[10:]:
    print(f't0 {r[0]:4d} nb {r[1]} gpu {r[2]:8.1f} ms  wall {r[3]:8.1f} ms  per update {r[2] / r[1]:6.1f}   [{r[4]}]')
