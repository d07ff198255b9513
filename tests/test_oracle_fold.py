"""Pins for the collective fold R (a9; R11) and the collective definitions.

R: widen to fp32, acc = x0, acc = fl32(acc + xk) in rank order, one RNE
rounding back, NaN -> canonical NaN.  Pinned against numpy float32 sequential
adds and torch's RNE bf16 / numpy's f16 conversions (independent libraries),
SPEC S:470-473, and a special-value table (-0, Inf - Inf, denormals)."""
import numpy as np
import pytest
import torch

import synth

BF16, F16, F32 = 0, 1, 2


def _to_f32(bits, dtype):
    if dtype == BF16:
        return (bits.astype(np.uint32) << 16).view(np.float32)
    if dtype == F16:
        return bits.view(np.float16).astype(np.float32)
    return bits.view(np.float32)


def _from_f32(v, dtype):
    if dtype == BF16:
        out = torch.from_numpy(v.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16).copy()
        out[np.isnan(v)] = 0x7FFF
    elif dtype == F16:
        with np.errstate(over="ignore"):
            out = v.astype(np.float16).view(np.uint16).copy()
        out[np.isnan(v)] = 0x7FFF
    else:
        out = v.view(np.uint32).copy()
        out[np.isnan(v)] = 0x7FFFFFFF
    return out


def _numpy_fold(inputs, dtype):
    acc = _to_f32(inputs[0], dtype).copy()
    with np.errstate(invalid="ignore", over="ignore"):
        for x in inputs[1:]:
            acc = (acc + _to_f32(x, dtype)).astype(np.float32)
    return _from_f32(acc, dtype)


def test_spec_example(orc):
    one, two, three = (np.array([b], np.uint16) for b in (0x3F80, 0x4000, 0x4040))   # bf16 1,2,3
    assert orc.reduce_sum(BF16, [one, two, three])[0] == 0x40C0                        # 6.0
    assert orc.reduce_sum(BF16, [one, two])[0] == 0x4040                               # 3.0


@pytest.mark.parametrize("dtype", [BF16, F16, F32])
@pytest.mark.parametrize("nranks", [2, 3, 4, 8])
def test_fold_matches_numpy_sequential(orc, dtype, nranks):
    n = 50_000
    ins = [synth.special_mix(n, 10 * nranks + r, dtype) if r == 1 else synth.normal(n, 3.0, r, dtype)
           for r in range(nranks)]
    assert np.array_equal(orc.reduce_sum(dtype, ins), _numpy_fold(ins, dtype))


def test_special_values(orc):
    d = BF16
    f = lambda *b: [np.array([x], np.uint16) for x in b]
    assert orc.reduce_sum(d, f(0x8000, 0x8000))[0] == 0x8000     # -0 + -0 = -0 (acc = x0, not 0 + x0)
    assert orc.reduce_sum(d, f(0x0000, 0x8000))[0] == 0x0000     # +0 + -0 = +0
    assert orc.reduce_sum(d, f(0x7F80, 0xFF80))[0] == 0x7FFF     # Inf - Inf -> canonical NaN
    assert orc.reduce_sum(d, f(0x7FC1, 0x3F80))[0] == 0x7FFF     # NaN payload -> canonical
    assert orc.reduce_sum(d, f(0x0001, 0x0001))[0] == 0x0002     # denormals kept (no FTZ/DAZ)
    assert orc.reduce_sum(d, f(0x7F7F, 0x7F7F))[0] == 0x7F80     # overflow -> +Inf
    assert orc.reduce_sum(F32, [np.array([1], np.uint32), np.array([1], np.uint32)])[0] == 2
    assert orc.reduce_sum(F16, [np.array([0x0001], np.uint16)] * 2)[0] == 0x0002
    assert orc.reduce_sum(F16, [np.array([0x7BFF], np.uint16)] * 2)[0] == 0x7C00


def test_rounding_once_not_per_step(orc):
    """Three bf16 values whose pairwise sums would round differently if the
    accumulator were rounded to bf16 after every add."""
    a = np.array([0x3F80], np.uint16)            # 1.0
    b = np.array([0x3B80], np.uint16)            # 2^-8 (half an ulp of 1.0 in bf16)
    out = orc.reduce_sum(BF16, [a, b, b])        # 1 + 2^-8 + 2^-8 = 1 + 2^-7 exactly
    assert out[0] == 0x3F81
    assert _numpy_fold([a, b, b], BF16)[0] == 0x3F81


def test_order_sensitive(orc):
    """permuting rank inputs can change low-order bits."""
    n = 20_000
    ins = [synth.normal(n, 10.0 ** (r - 2), r, F32) for r in range(4)]
    a = orc.reduce_sum(F32, ins)
    b = orc.reduce_sum(F32, ins[::-1])
    assert not np.array_equal(a, b)


def test_collective_definitions(orc):
    """AG concatenates, RS gives rank r the fold of shard r, AR = fold; and
    transparency: folding decompressed inputs == folding the originals."""
    N, n = 4, 4096 * 4
    ins = [synth.normal(n, 0.02, r) for r in range(N)]
    ag = orc.allgather(BF16, ins)
    assert np.array_equal(ag.reshape(N, n), np.stack(ins))
    rs = orc.reduce_scatter(BF16, ins, N)
    ar = orc.allreduce(BF16, ins)
    assert np.array_equal(np.concatenate(rs), ar)
    dec = [orc.decompress(orc.compress(BF16, x), n, BF16)[1] for x in ins]
    assert np.array_equal(orc.allreduce(BF16, dec), ar)
