"""Pins for the oracle's split/join (a1).

The pins are independent of the oracle's own formulas: worked examples from
SPEC, an exhaustive bijection over every 16-bit pattern, and the meaning of
the fields checked against numpy's frexp/signbit (the exponent field IS the
binary exponent of the value)."""
import numpy as np
import pytest

BF16, F16, F32 = 0, 1, 2


def test_spec_worked_examples(orc):
    # SPEC S:61 bf16 1.0 = 0x3F80 -> symbol 0x7F, residual 0x00
    s, r = orc.split(BF16, np.array([0x3F80], np.uint16))
    assert (s[0], r[0]) == (0x7F, 0x00)
    # SPEC S:62 bf16 -1.5 = 0xBFC0 -> symbol 0x7F, residual 0xC0
    s, r = orc.split(BF16, np.array([0xBFC0], np.uint16))
    assert (s[0], r[0]) == (0x7F, 0xC0)
    # SPEC S:64 f16 1.0 = 0x3C00 -> symbol 0x3C, residual 0x00
    s, r = orc.split(F16, np.array([0x3C00], np.uint16))
    assert (s[0], r[0]) == (0x3C, 0x00)
    # SPEC S:73 inverse
    assert orc.join(BF16, np.array([0x7F], np.uint8), np.array([0], np.uint32))[0] == 0x3F80


@pytest.mark.parametrize("dtype", [BF16, F16])
def test_exhaustive_bijection_16bit(orc, dtype):
    allbits = np.arange(1 << 16, dtype=np.uint16)
    s, r = orc.split(dtype, allbits)
    assert np.array_equal(orc.join(dtype, s, r), allbits)
    # injective: the (symbol, residual) pairs are all distinct and cover 2^16
    key = s.astype(np.uint32) << 8 | r
    assert np.unique(key).size == 1 << 16
    assert r.max() < 256


def _frexp_fields(vals):
    m, e = np.frexp(np.abs(vals))
    return m, e


def test_bf16_symbol_is_binary_exponent(orc):
    allbits = np.arange(1 << 16, dtype=np.uint16)
    s, r = orc.split(BF16, allbits)
    vals = (allbits.astype(np.uint32) << 16).view(np.float32)
    finite = np.isfinite(vals) & (vals != 0)
    normal = finite & (np.abs(vals) >= np.float32(2.0 ** -126))
    m, e = _frexp_fields(vals[normal].astype(np.float64))
    # |v| = m * 2^e, m in [0.5, 1)  =>  biased exponent = e - 1 + 127
    assert np.array_equal(s[normal].astype(np.int64), e - 1 + 127)
    # fraction bits: (2m - 1) * 2^7, sign bit in residual bit 7
    assert np.array_equal(r[normal] & 0x7F, ((2 * m - 1) * 128).astype(np.int64))
    assert np.array_equal(r[finite] >> 7, np.signbit(vals[finite]).astype(np.uint32))
    # zeros, subnormals have exponent field 0; Inf/NaN 255
    assert np.all(s[~np.isfinite(vals)] == 255)
    assert np.all(s[finite & ~normal] == 0)


def test_f16_symbol_is_sign_exponent_two_msbs(orc):
    allbits = np.arange(1 << 16, dtype=np.uint16)
    s, r = orc.split(F16, allbits)
    vals = allbits.view(np.float16).astype(np.float64)
    normal = np.isfinite(vals) & (np.abs(vals) >= 2.0 ** -14)
    m, e = _frexp_fields(vals[normal])
    assert np.array_equal((s[normal] >> 2) & 0x1F, e - 1 + 15)          # 5 exponent bits
    assert np.array_equal(s[normal] >> 7, np.signbit(vals[normal]))
    mant10 = ((2 * m - 1) * 1024).astype(np.int64)
    assert np.array_equal(((s[normal] & 3).astype(np.int64) << 8) | r[normal], mant10)


def test_f32_split_fields_and_roundtrip(orc):
    rng = np.random.default_rng(3)
    bits = rng.integers(0, 1 << 32, size=200_000, dtype=np.uint64).astype(np.uint32)
    bits[:8] = [0, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00001, 1, 0x3F800000, 0xC0490FDB]
    s, r = orc.split(F32, bits)
    assert np.array_equal(orc.join(F32, s, r), bits)
    vals = bits.view(np.float32).astype(np.float64)
    normal = np.isfinite(vals) & (np.abs(vals) >= 2.0 ** -126)
    m, e = _frexp_fields(vals[normal])
    assert np.array_equal(s[normal].astype(np.int64), e - 1 + 127)
    frac23 = ((2 * m - 1) * (1 << 23)).astype(np.int64)
    lo16 = r[normal] & 0xFFFF
    hi8 = r[normal] >> 16
    assert np.array_equal(((hi8 & 0x7F).astype(np.int64) << 16) | lo16, frac23)
    assert np.array_equal(hi8 >> 7, np.signbit(vals[normal]))


@pytest.mark.parametrize("dtype,frac", [(BF16, 0.5), (F16, 0.5), (F32, 0.75)])
def test_residual_fraction_of_stream(orc, dtype, frac):
    """the uncompressed part is ~1/2 (bf16) and ~3/4 (fp32) of the bytes."""
    import synth
    n = 4096 * 8
    bits = synth.uniform(n, 1, dtype)
    st = orc.sections(orc.compress(dtype, bits))
    res_bytes = st["off_tab"] - st["off_res0"]
    assert res_bytes == frac * n * orc.ELEM_BYTES[dtype]
