"""CPU-side checks: the C-ABI library loads and exports every declared symbol,
the Python mirror validates arguments like the reference, and the input
generators produce the BASELINE shapes.  No kernel is launched here."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import REPO

HEADER = os.path.join(REPO, "include", "strom_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(strom_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1910_01260_b200 import _capi

    names = declared_functions()
    assert len(names) >= 17
    missing = [n for n in names if not hasattr(_capi.lib, n)]
    assert not missing, missing
    # and the Python binding types every one of them
    assert set(names) <= set(_capi.EXPORTED)


def test_abi_version_matches_header():
    from paper_1910_01260_b200 import _capi

    m = re.search(r"#define STROM_B200_ABI_VERSION (\d+)", open(HEADER).read())
    assert _capi.lib.strom_abi_version() == int(m.group(1))


def test_library_is_sm100a_only():
    """The shipped .so carries sm_100a SASS (cuobjdump) and DMMA for the fp64 contractions."""
    import shutil
    import subprocess

    from paper_1910_01260_b200 import _capi

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([tool, "-sass", _capi.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA" in sass


def test_error_codes_map_to_reference_exceptions():
    from paper_1910_01260_b200 import _capi, errors

    with pytest.raises(ValueError):
        _capi.check(1)
    with pytest.raises(errors.SingularMatrixError):
        _capi.check(4)
    with pytest.raises(errors.BasisError):
        _capi.check(5)


def test_api_argument_validation_without_gpu():
    from paper_1910_01260_b200 import TimeGrid, basis

    with pytest.raises(ValueError):
        basis.isvd_init(np.ones(3), 1e-8, cap_mode="drop")
    with pytest.raises(ValueError):
        TimeGrid(np.array([0.1, -0.1]))
    with pytest.raises(ValueError):
        TimeGrid(np.array([]))
    assert TimeGrid.uniform(0.5, 4).total_time == 2.0


def test_lds_validation():
    import scipy.sparse as sp

    from paper_1910_01260_b200 import LinearDynamicalSystem

    with pytest.raises(ValueError):
        LinearDynamicalSystem(a=sp.eye(3), b=sp.csr_array((4, 1)), c=np.ones((3, 1)), x0=np.zeros(3),
                              input_signal=lambda k: np.zeros(1))


def test_cfg4_operator_structure():
    from paper_1910_01260_b200 import workloads as wl

    a = wl.cfg4_operator(nx=12)
    assert a.nnz == 7 * 12**3 - 6 * 12**2
    assert a.indices.dtype == np.int32
    # upwind + diffusion: strictly diagonally dominant rows with negative diagonal
    d = a.diagonal()
    off = np.asarray(abs(a).sum(axis=1)).ravel() - np.abs(d)
    assert np.all(d < 0) and np.all(np.abs(d) >= off * (1 - 1e-12))


def test_cfg1_system_is_periodic_mass_conserving():
    from paper_1910_01260_b200 import workloads as wl

    d = wl.cfg1_system(0.02, n=64)
    # periodic upwind + central diffusion: columns sum to zero (mass conservation)
    assert np.max(np.abs(np.asarray(d.a.sum(axis=0)).ravel())) <= 1e-9 * abs(d.a).max()


def test_cfg2_generator_shapes():
    from paper_1910_01260_b200 import workloads as wl

    x, q, w, s = wl.cfg2_stream_numpy(n=512, cols=80, rank=8)
    assert x.shape == (512, 80) and x.flags.f_contiguous
    assert np.allclose(q.T @ q, np.eye(8), atol=1e-12)
    assert np.allclose(s, 10.0 ** (-np.arange(8) / 8))
