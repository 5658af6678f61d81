"""SPTN reader/writer (paper_2605_17633_b200.sptn) against the reference format (tensor.py:65-116,
grid.py:122-136): the reference's own format tests (test_tensor.py:28-103) restated, plus files the
reference wrote (tests/golden/sptn/, tests/golden/make_golden.py sptn_files)."""

import struct
import sys
from pathlib import Path

import numpy as np
import pytest

from paper_2605_17633_b200 import sptn
from paper_2605_17633_b200.sptn import (SptnBadDtype, SptnBadMagic, SptnBadShape, SptnBadVersion, SptnTruncated,
                                        tensor_read, tensor_write)

GOLD = Path(__file__).resolve().parent / "golden" / "sptn"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from oracle import zs_oracle as O  # noqa: E402


def test_header_layout_scalar_shaped(tmp_path):  # test_tensor.py:31-43
    path = tmp_path / "one.sptn"
    tensor_write(np.array([3.0], dtype=np.float32), path)
    raw = path.read_bytes()
    assert len(raw) == 18 + 4
    assert raw[:4] == b"SPTN" and raw[4] == 1 and raw[5] == 0 and raw[6] == 1
    assert raw[7:10] == b"\x00\x00\x00"
    assert struct.unpack("<Q", raw[10:18]) == (1,)
    assert struct.unpack("<f", raw[18:]) == (3.0,)


def test_roundtrip_random(tmp_path):  # test_tensor.py:52-62
    rng = np.random.default_rng(20240817)
    path = tmp_path / "t.sptn"
    for _ in range(200):
        shape = tuple(int(rng.integers(1, 6)) for _ in range(int(rng.integers(1, 5))))
        t = rng.standard_normal(shape).astype(np.float32)
        tensor_write(t, path)
        back = tensor_read(path)
        assert back.shape == t.shape and back.dtype == np.float32
        assert np.array_equal(back, t)


def test_torch_tensor_write_and_device_read(tmp_path):
    torch = pytest.importorskip("torch")
    t = torch.arange(12, dtype=torch.float32).reshape(3, 4)
    tensor_write(t, tmp_path / "t.sptn")
    back = tensor_read(tmp_path / "t.sptn", device="cpu")
    assert isinstance(back, torch.Tensor) and torch.equal(back, t)
    with pytest.raises(TypeError):
        tensor_write(t.double(), tmp_path / "d.sptn")


@pytest.mark.parametrize("raw, exc", [
    (b"XXXX" + bytes(20), SptnBadMagic),
    (b"SPTN" + bytes([9, 0, 1]) + bytes(3) + struct.pack("<Q", 1) + bytes(4), SptnBadVersion),
    (b"SPTN" + bytes([1, 7, 1]) + bytes(3) + struct.pack("<Q", 1) + bytes(4), SptnBadDtype),
    (b"SPTN" + bytes([1, 0, 0]) + bytes(3), SptnBadShape),
    (b"SPTN\x01\x00", SptnTruncated),
    (b"SPTN" + bytes([1, 0, 2]) + bytes(3) + struct.pack("<Q", 1), SptnTruncated),
    (b"SPTN" + bytes([1, 0, 1]) + bytes(3) + struct.pack("<Q", 0), SptnBadShape),
])
def test_malformed_files(tmp_path, raw, exc):  # test_tensor.py:64-97
    path = tmp_path / "bad.sptn"
    path.write_bytes(raw)
    with pytest.raises(exc):
        tensor_read(path)
    assert issubclass(exc, ValueError)


def test_truncated_payload_and_trailing_bytes(tmp_path):
    path = tmp_path / "s.sptn"
    tensor_write(np.arange(6, dtype=np.float32).reshape(2, 3), path)
    raw = path.read_bytes()
    path.write_bytes(raw[:-4])
    with pytest.raises(SptnTruncated):
        tensor_read(path)
    path.write_bytes(raw + b"\x00")
    with pytest.raises(SptnBadShape):
        tensor_read(path)


def test_zero_extent_and_missing_file(tmp_path):
    with pytest.raises(SptnBadShape):
        tensor_write(np.zeros((0, 3), dtype=np.float32), tmp_path / "e.sptn")
    with pytest.raises(OSError):
        tensor_read(tmp_path / "nope.sptn")


def test_reference_written_files_read_and_rewrite_bit_exact(tmp_path):
    for f in sorted(GOLD.glob("*.sptn")):
        t = tensor_read(f)
        tensor_write(t, tmp_path / f.name)
        assert (tmp_path / f.name).read_bytes() == f.read_bytes(), f.name
    assert np.array_equal(tensor_read(GOLD / "scalar.sptn"), np.array([3.0], np.float32))
    # the reference's Rng(7).normal((3, 5, 4)) == the oracle's splitmix restatement
    assert np.array_equal(tensor_read(GOLD / "rank3.sptn"), O.SplitMix(7).normal((3, 5, 4)))
    # Sobel map written by the reference == the oracle's restatement, bit for bit
    x = O.SplitMix(1).normal((6, 10, 8))
    assert np.array_equal(tensor_read(GOLD / "sobel_6x10.sptn"), O.sobel_magnitude(x))


def test_permutation_files(tmp_path):
    p = sptn.permutation_read(GOLD / "morton_6x10.sptn")
    assert np.array_equal(p.forward, O.morton_order(6, 10))
    sptn.permutation_write(p, tmp_path / "m.sptn")
    assert (tmp_path / "m.sptn").read_bytes() == (GOLD / "morton_6x10.sptn").read_bytes()
    tensor_write(np.array([0.0, 1.5], np.float32), tmp_path / "frac.sptn")
    with pytest.raises(ValueError):
        sptn.permutation_read(tmp_path / "frac.sptn")
    tensor_write(np.zeros((2, 2), np.float32), tmp_path / "r2.sptn")
    with pytest.raises(ValueError):
        sptn.permutation_read(tmp_path / "r2.sptn")
