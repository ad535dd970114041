"""Time the compaction of a cfg2 state (diagnostics)."""
import sys
import time

import torch

sys.path.insert(0, '.')
from paper_1910_01260_b200 import _capi, basis, workloads as wl  # noqa: E402

xt, _, _, _ = wl.cfg2_stream_torch(n=1 << 20, cols=260, rank=64, seed=0)
st = basis.isvd_init(xt[0], 1e-9, tol_sv=1e-9, r_max=64, cap_mode='truncate')
st = basis.ingest_simulation(st, xt[1:100].T)
torch.cuda.synchronize()
lib = _capi.lib
lib.strom_profile_reset()
lib.strom_profile_enable(1)
st2 = basis.ingest_simulation(st, xt[100:260].T)
torch.cuda.synchronize()
lib.strom_profile_enable(0)
pl = (_capi.i64 * 16)(); pms = (_capi.dbl * 16)(); pby = (_capi.dbl * 16)()
lib.strom_profile_read(16, pl, pms, pby)
names = ["pass", "second", "decide", "step_b", "v_update", "compact_prep", "compact_pass", "spatial", "st_gemm",
         "st_small", "lu", "temporal", "other"]
for k in range(13):
    if pl[k]:
        print(f"{names[k]:14s} launches {pl[k]:5d}  ms {pms[k]:9.3f}  mean_us {1e3 * pms[k] / pl[k]:8.1f}")
print('rank', st2.rank, 'sigma0', float(st2.sigma[0]))
