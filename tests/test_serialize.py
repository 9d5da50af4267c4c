"""CPU: bit-exact range / snapshot serialization (reference module `serialize`,
SPEC.md:466-519), every example of its spec."""
import numpy as np
import pytest

from paper_2503_13795_b200 import serialize as ser
from paper_2503_13795_b200 import TgError


def _payloads(dtype):
    """Random values plus -0.0, subnormals, +-inf and NaNs with payloads."""
    rng = np.random.default_rng(3)
    a = rng.standard_normal(64).astype(dtype)
    ib = np.int64 if dtype == np.float64 else np.int32
    special_bits = ([0x8000000000000000, 0x0000000000000001, 0x7FF0000000000000, 0xFFF0000000000000,
                     0x7FF8000000000123, 0xFFF4000000000abc] if dtype == np.float64 else
                    [0x80000000, 0x00000001, 0x7F800000, 0xFF800000, 0x7FC00123, 0xFFA00abc])
    sp = np.array(special_bits, dtype=np.uint64 if dtype == np.float64 else np.uint32).view(dtype)
    return np.concatenate([a, sp])


def test_seven_fp64_values_are_56_bytes():
    v = np.arange(7, dtype=np.float64)
    b = ser.save_range(v)
    assert len(b) == 56                       # PAPER Table 4, "Raw payload size: 56 bytes"
    assert b == v.astype("<f8").tobytes()     # headerless little-endian


def test_empty_range_and_fp32_with_grads_sizes():
    assert ser.save_range(np.zeros(0)) == b""
    v = np.ones(3, np.float32)
    assert len(ser.save_range(v, np.zeros(3, np.float32))) == 24   # 3 * 4 * 2


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_round_trip_is_bit_exact(dtype):
    v, g = _payloads(dtype), _payloads(dtype)[::-1].copy()
    b = ser.save_range(v, g)
    v2, g2 = np.zeros_like(v), np.zeros_like(g)
    ser.load_range(b, v2, g2)
    ib = np.uint64 if dtype == np.float64 else np.uint32
    np.testing.assert_array_equal(v.view(ib), v2.view(ib))
    np.testing.assert_array_equal(g.view(ib), g2.view(ib))


def test_short_or_cross_precision_load_is_format_error_without_partial_write():
    v = np.arange(7, dtype=np.float64)
    b = ser.save_range(v)
    dst = np.full(7, 9.0)
    with pytest.raises(TgError, match="TG_FORMAT"):
        ser.load_range(b[:55], dst)           # 55 bytes where 56 expected
    np.testing.assert_array_equal(dst, 9.0)   # nothing applied
    b32 = ser.save_range(v.astype(np.float32))
    with pytest.raises(TgError, match="TG_FORMAT"):
        ser.load_range(b32, dst)              # fp32 payload into an fp64 range
    np.testing.assert_array_equal(dst, 9.0)


def test_snapshot_header_round_trip_and_errors():
    assert len(ser.save_snapshot(np.zeros(0))) == 18      # header only: 4 + 4 + 1 + 1 + 8
    v, g = _payloads(np.float64), _payloads(np.float64)[::-1].copy()
    s = ser.save_snapshot(v, g)
    assert s[:4] == b"BTSG" and s[4:8] == (1).to_bytes(4, "little") and s[8] == 1 and s[9] == 1
    assert int.from_bytes(s[10:18], "little") == v.size
    v2, g2 = np.zeros_like(v), np.zeros_like(g)
    assert ser.load_snapshot(s, v2, g2) == {"dtype": "f64", "count": v.size, "grads": True}
    np.testing.assert_array_equal(v.view(np.uint64), v2.view(np.uint64))
    np.testing.assert_array_equal(g.view(np.uint64), g2.view(np.uint64))
    with pytest.raises(TgError, match="TG_FORMAT"):
        ser.load_snapshot(s[:10], v2)         # truncated header
    with pytest.raises(TgError, match="TG_FORMAT"):
        ser.load_snapshot(b"XXXX" + s[4:], v2)
    with pytest.raises(TgError, match="TG_FORMAT"):
        ser.load_snapshot(s[:4] + (2).to_bytes(4, "little") + s[8:], v2)   # unsupported version
    with pytest.raises(TgError, match="TG_CAPACITY"):
        ser.load_snapshot(s, np.zeros(3))


def test_cross_precision_snapshot_is_format_error_without_partial_write():
    """An fp64 snapshot loaded into an fp32 range (and the reverse) is
    TG_FORMAT before any byte is written: the range and a guard region past
    it keep their contents (all-or-nothing loads)."""
    v = np.arange(4, dtype=np.float64) + 0.5
    s64 = ser.save_snapshot(v)
    buf = np.full(8, 7.0, np.float32)
    with pytest.raises(TgError, match="TG_FORMAT"):
        ser.load_snapshot(s64, buf[:4])
    np.testing.assert_array_equal(buf, 7.0)
    s32 = ser.save_snapshot(v.astype(np.float32))
    buf64 = np.full(8, 7.0)
    with pytest.raises(TgError, match="TG_FORMAT"):
        ser.load_snapshot(s32, buf64[:4])
    np.testing.assert_array_equal(buf64, 7.0)
    assert ser.load_snapshot(s32, buf[:4])["count"] == 4
    np.testing.assert_array_equal(buf[:4], v.astype(np.float32))
    np.testing.assert_array_equal(buf[4:], 7.0)
