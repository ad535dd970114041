"""STROMMAT files (reference persist.py, tests mirror pkg/tests/test_persist.py)
and the device save/load path of pipeline.py:127-176."""

import numpy as np
import pytest

from paper_1910_01260_b200 import persist


def test_one_by_one_layout(tmp_path):
    path = tmp_path / "m.strommat"
    persist.write_matrix(path, np.array([[0.0]]))
    blob = path.read_bytes()
    assert len(blob) == persist.HEADER_SIZE + 8
    assert blob[:8] == b"STROMMAT"
    assert blob[persist.HEADER_SIZE:] == b"\x00" * 8


def test_header_fields(tmp_path):
    path = tmp_path / "m.strommat"
    persist.write_matrix(path, np.ones((3, 2)))
    blob = path.read_bytes()
    assert int.from_bytes(blob[8:12], "little") == 1
    assert int.from_bytes(blob[12:20], "little") == 3 and int.from_bytes(blob[20:28], "little") == 2


@pytest.mark.parametrize("bad", [np.empty((0, 0)), np.array([[np.inf]]), np.array([[1.0, np.nan]])])
def test_rejected_on_write(tmp_path, bad):
    with pytest.raises(persist.MatrixFileError):
        persist.write_matrix(tmp_path / "e.strommat", bad)


def test_roundtrip_bit_identity_many_shapes(tmp_path):
    rng = np.random.default_rng(1)
    path = tmp_path / "m.strommat"
    for _ in range(30):
        m = rng.standard_normal((int(rng.integers(1, 30)), int(rng.integers(1, 30))))
        persist.write_matrix(path, m)
        back = persist.read_matrix(path)
        assert back.flags.c_contiguous and back.tobytes() == m.tobytes()


def test_column_major_payload_and_vector(tmp_path):
    m = np.array([[1.0, 3.0], [2.0, 4.0]])
    path = tmp_path / "m.strommat"
    persist.write_matrix(path, m)
    payload = np.frombuffer(path.read_bytes()[persist.HEADER_SIZE:], dtype="<f8")
    np.testing.assert_array_equal(payload, [1.0, 2.0, 3.0, 4.0])
    persist.write_matrix(path, np.array([1.0, 2.0]))
    assert persist.read_matrix(path).shape == (2, 1)


@pytest.mark.parametrize(
    "mangle",
    [
        lambda blob: b"WRONGMAG" + blob[8:],
        lambda blob: blob[:8] + b"\x02\x00\x00\x00" + blob[12:],
        lambda blob: blob[: persist.HEADER_SIZE - 4],
        lambda blob: blob[:-1],
        lambda blob: blob + b"\x00",
        lambda blob: blob[: persist.HEADER_SIZE],
        lambda blob: blob[:12] + (0).to_bytes(8, "little") + blob[20:],
    ],
    ids=["magic", "version", "short-header", "truncated", "padded", "no-payload", "zero-rows"],
)
def test_corruption_detected(tmp_path, mangle):
    path = tmp_path / "m.strommat"
    persist.write_matrix(path, np.arange(6.0).reshape(2, 3) + 1.0)
    path.write_bytes(mangle(path.read_bytes()))
    with pytest.raises(persist.MatrixFileError):
        persist.read_matrix(path)


def test_nonfinite_payload_rejected_on_read(tmp_path):
    path = tmp_path / "m.strommat"
    persist.write_matrix(path, np.ones((1, 2)))
    blob = path.read_bytes()
    path.write_bytes(blob[:-8] + np.array([np.nan]).tobytes())
    with pytest.raises(persist.MatrixFileError, match="non-finite"):
        persist.read_matrix(path)


def test_cpu_tensor_roundtrip(tmp_path):
    import torch

    m = torch.arange(12, dtype=torch.float64).reshape(3, 4)
    path = tmp_path / "t.strommat"
    for t in (m, m.T.contiguous().T):  # row-major and column-major layouts
        persist.write_matrix(path, t)
        assert persist.read_matrix(path).tobytes() == m.numpy().tobytes()


@pytest.mark.gpu
def test_device_roundtrip_and_basis_files(cuda, tmp_path):
    import torch

    from paper_1910_01260_b200 import basis, workloads as wl

    rng = np.random.default_rng(3)
    m = rng.standard_normal((37, 5))
    dm = torch.as_tensor(m, device="cuda")
    path = tmp_path / "d.strommat"
    persist.write_matrix(path, dm)
    assert persist.read_matrix(path).tobytes() == m.tobytes()
    back = persist.read_matrix_device(path)
    assert back.is_cuda and back.stride(0) == 1 and torch.equal(back.cpu(), dm.cpu())
    with pytest.raises(persist.MatrixFileError):
        persist.write_matrix(path, torch.tensor([[float("inf")]], device="cuda"))
    # save_bases / load_basis round trip of a trained state
    x, _, _, _ = wl.cfg2_stream_numpy(n=256, cols=24, rank=6, seed=2, decades_per=3.0)
    st = basis.ingest_simulation(basis.isvd_init(x[:, 0], 1e-10), x[:, 1:])
    bs = basis.build_basis_set(st, 4, 2, 8, 3)
    names = persist.save_bases(st, bs, tmp_path / "b")
    assert names[0] == "phi_s.strommat" and names[-1] == "v.strommat" and len(names) == 1 + 4 + 2
    lb = persist.load_basis(tmp_path / "b")
    assert torch.equal(lb.phi_s.cpu(), bs.phi_s.cpu()) and lb.n_mu == 3
    assert all(torch.equal(a.cpu(), b.cpu()) for a, b in zip(lb.temporal, bs.temporal))
    sl = persist.load_basis(tmp_path / "b", n_s=2, n_t=1)
    assert sl.phi_s.shape == (256, 2) and sl.temporal[0].shape == (8, 1)
    with pytest.raises(ValueError):
        persist.load_basis(tmp_path / "b", n_s=5)
    with pytest.raises(FileNotFoundError):
        persist.load_basis(tmp_path / "nothing")


def test_reference_written_file_bit_exact(tmp_path):
    """Bytes written by the reference (tests/golden/make_golden.py gen_persist) read back
    exactly, and this writer reproduces them byte for byte."""
    import os

    gdir = os.path.join(os.path.dirname(__file__), "golden")
    ref_path = os.path.join(gdir, "golden_ref_5x3.strommat")
    m = np.load(os.path.join(gdir, "golden_ref_5x3_values.npy"))
    assert persist.read_matrix(ref_path).tobytes() == m.tobytes()
    path = tmp_path / "mine.strommat"
    persist.write_matrix(path, m)
    assert path.read_bytes() == open(ref_path, "rb").read()
