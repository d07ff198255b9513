"""Oracle pins for the min / max folds (§3.4 P:402 "sum, min, or max"; R25).

R25: IEEE 754-2019 minimum / maximum applied in rank order -- a NaN operand makes the result NaN
(canonical on output, like the sum), -0 < +0, otherwise the smaller / larger value; the result is
one of the inputs, so the output rounding is exact.  Pinned by: numpy's reductions on NaN- and
zero-free inputs (bit-exact), a hand-written special-value table, and order invariance (min and
max, unlike the fp32 sum, do not depend on the rank order).
"""
import numpy as np
import pytest
import torch

import synth

BF16, F16, F32 = 0, 1, 2
MIN, MAX = 1, 2
NPF = {F16: np.float16, F32: np.float32}


def as_float(dtype, bits):
    if dtype == BF16:
        return (bits.astype(np.uint32) << 16).view(np.float32)
    return bits.view(NPF[dtype]).astype(np.float32)


@pytest.mark.parametrize("dtype", [BF16, F16, F32])
@pytest.mark.parametrize("op", [MIN, MAX])
@pytest.mark.parametrize("nranks", [2, 3, 8])
def test_minmax_matches_numpy_on_ordinary_values(orc, dtype, op, nranks):
    ins = [synth.normal(5000, 1.0, 10 * nranks + r, dtype) for r in range(nranks)]
    ins = [np.where(b & (0x7FFFFFFF if dtype == F32 else 0x7FFF) == 0, b | 1, b) for b in ins]  # no zeros
    got = orc.reduce(dtype, ins, op)
    vals = np.stack([as_float(dtype, b) for b in ins])
    ref = vals.min(0) if op == MIN else vals.max(0)
    assert np.array_equal(as_float(dtype, got), ref)
    # the result is one of the inputs, bit for bit
    assert all(any(got[i] == b[i] for b in ins) for i in range(0, 5000, 97))


@pytest.mark.parametrize("op", [MIN, MAX])
def test_minmax_is_independent_of_rank_order(orc, op):
    ins = [synth.special_mix(3000, 50 + r, BF16) for r in range(5)]
    ref = orc.reduce(BF16, ins, op)
    rng = np.random.default_rng(3)
    for _ in range(4):
        perm = rng.permutation(5)
        assert np.array_equal(orc.reduce(BF16, [ins[k] for k in perm], op), ref)


def test_minmax_special_value_table(orc):
    z, nz, inf, ninf, nan, one, m1 = 0x0000, 0x8000, 0x7F80, 0xFF80, 0x7FC1, 0x3F80, 0xBF80
    cases = [  # (a, b, min, max) in bf16 bits
        (z, nz, nz, z), (nz, z, nz, z), (z, z, z, z), (nz, nz, nz, nz),
        (inf, one, one, inf), (ninf, one, ninf, one), (inf, ninf, ninf, inf),
        (nan, one, 0x7FFF, 0x7FFF), (one, nan, 0x7FFF, 0x7FFF), (nan, nan, 0x7FFF, 0x7FFF),
        (one, m1, m1, one), (m1, nz, m1, nz),
    ]
    a = np.array([c[0] for c in cases], np.uint16)
    b = np.array([c[1] for c in cases], np.uint16)
    assert orc.reduce(BF16, [a, b], MIN).tolist() == [c[2] for c in cases]
    assert orc.reduce(BF16, [a, b], MAX).tolist() == [c[3] for c in cases]
    # f32: same rules, canonical NaN 0x7FFFFFFF
    f = np.array([0x00000000, 0x80000000, 0x7FC00001], np.uint32)
    g = np.array([0x80000000, 0x00000000, 0x3F800000], np.uint32)
    assert orc.reduce(F32, [f, g], MIN).tolist() == [0x80000000, 0x80000000, 0x7FFFFFFF]
    assert orc.reduce(F32, [f, g], MAX).tolist() == [0x00000000, 0x00000000, 0x7FFFFFFF]


def test_sum_op_is_the_pinned_fold(orc):
    ins = [synth.normal(4096, 0.02, 60 + r, BF16) for r in range(4)]
    assert np.array_equal(orc.reduce(BF16, ins, 0), orc.reduce_sum(BF16, ins))
