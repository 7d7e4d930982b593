"""DMAT files (reference io suite, tests/test_io.cpp; layout dmat.hpp:10-19): host round
trip and the reference's error contract (IoError with byte offsets) — no GPU needed."""
import numpy as np
import pytest

from paper_2110_03423_b200.dmat import IoError, read_dmat, write_dmat


def test_round_trip_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    a = rng.standard_normal((37, 11))
    a[3, 4] = -0.0
    a[5, 6] = 1e-310  # subnormal
    p = str(tmp_path / "a.dmat")
    write_dmat(p, a)
    raw = open(p, "rb").read()
    assert raw[:6] == b"DMAT1\n" and len(raw) == 22 + a.size * 8
    assert int.from_bytes(raw[6:14], "little") == 37 and int.from_bytes(raw[14:22], "little") == 11
    b = read_dmat(p)
    assert b.tobytes() == a.astype("<f8").tobytes()


def test_errors_carry_offsets(tmp_path):
    p = str(tmp_path / "x.dmat")
    with pytest.raises(IoError):
        read_dmat(str(tmp_path / "missing.dmat"))
    open(p, "wb").write(b"DMAT2\n" + bytes(16))
    with pytest.raises(IoError) as e:
        read_dmat(p)
    assert e.value.offset == 0
    open(p, "wb").write(b"DMAT1\n" + bytes(10))
    with pytest.raises(IoError) as e:
        read_dmat(p)
    assert e.value.offset == 16
    open(p, "wb").write(b"DMAT1\n" + (0).to_bytes(8, "little") + (3).to_bytes(8, "little"))
    with pytest.raises(IoError) as e:
        read_dmat(p)
    assert e.value.offset == 6
    write_dmat(p, np.ones((2, 3)))
    raw = open(p, "rb").read()
    open(p, "wb").write(raw[:-5])
    with pytest.raises(IoError) as e:
        read_dmat(p)
    assert e.value.offset == len(raw) - 5
    open(p, "wb").write(raw + b"x")
    with pytest.raises(IoError) as e:
        read_dmat(p)
    assert e.value.offset == len(raw)
