"""Isolated fused-pass bandwidth over the live-column count c (diagnostics)."""
import ctypes as C
import sys

sys.path.insert(0, '.')
from paper_1910_01260_b200 import _capi  # noqa: E402

n = 1 << 20
for c in (64, 68, 72, 80, 88, 96):
    ms = C.c_double()
    rc = _capi.lib.strom_debug_pass_bw(n, c, 30, 1, C.byref(ms))
    assert rc == 0, _capi.lib.strom_last_error()
    gb = 8.0 * n * (c + 3) / (ms.value / 1e3) / 1e9
    print(f"c={c:4d} {ms.value * 1e3:8.1f} us  {gb:7.0f} GB/s", flush=True)
