"""Isolated fused-pass bandwidth: strom_debug_pass_bw over (c, reserve, dbg) (diagnostics)."""
import ctypes as C
import os
import sys

sys.path.insert(0, '.')
from paper_1910_01260_b200 import _capi  # noqa: E402

n = 1 << 20
for c in (16, 64, 96, 127):
    ms = C.c_double()
    rc = _capi.lib.strom_debug_pass_bw(n, c, 20, 1, C.byref(ms))
    assert rc == 0, _capi.lib.strom_last_error()
    gb = 8.0 * n * (c + 3) / (ms.value / 1e3) / 1e9
    print(f"dbg={os.environ.get('STROM_PASS_DBG', '0')} stage_kb={os.environ.get('STROM_STAGE_KB', '140')} "
          f"c={c:4d} {ms.value * 1e3:8.1f} us  {gb:7.0f} GB/s", flush=True)
