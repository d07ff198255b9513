"""Pins for the oracle's UZB1 stream (a1-a8, a11).

* losslessness over dtypes, distributions and edge sizes (SPEC S:77, S:250,
  S:564): n in {0, 1, B-1, B, B+1, kB+17}, multi-chunk, global-table mode;
* compression ratios against the Shannon bound computed in closed form from
  the value distribution (U: P(|v| in [2^k, 2^(k+1))) = 2^k; W/G: normal
  binade masses via erf) and against the paper's printed ratios (P:550,
  P:722, Table 1) with SPEC's tolerances;
* the empirical entropy oracle of SPEC S:156-164 / S:566;
* the stored-raw bound on incompressible input (R13);
* corrupt-stream and mismatch errors (O12)."""
import math

import numpy as np
import pytest

import synth

BF16, F16, F32 = 0, 1, 2
EB = {BF16: 2, F16: 2, F32: 4}
RES_BITS = {BF16: 8, F16: 8, F32: 24}


def _roundtrip(orc, dtype, bits, **kw):
    s = orc.compress(dtype, bits, **kw)
    st, out = orc.decompress(s, bits.size, dtype)
    assert st == orc.OK
    assert np.array_equal(out, bits)
    hd = orc.parse_header(s)
    assert hd["magic"] == b"UZB1" and hd["n"] == bits.size and hd["dtype"] == dtype
    assert hd["total_bytes"] == len(s)
    return s


@pytest.mark.parametrize("dtype", [BF16, F16, F32])
@pytest.mark.parametrize("n", [0, 1, 4095, 4096, 4097, 3 * 4096 + 17])
def test_roundtrip_edge_sizes(orc, dtype, n):
    for gen in (lambda: synth.normal(n, 0.02, n, dtype), lambda: synth.special_mix(n, n, dtype),
                lambda: synth.random_bits(n, n, dtype), lambda: synth.constant(n, 0, dtype)):
        _roundtrip(orc, dtype, gen())


@pytest.mark.parametrize("dtype", [BF16, F16, F32])
def test_roundtrip_multichunk_and_global(orc, dtype):
    n = 4096 * 37 + 5
    bits = synth.normal(n, 0.02, 7, dtype)
    bits[4096 * 20:4096 * 21] = synth.random_bits(4096, 8, dtype)       # one incompressible block
    s_local = _roundtrip(orc, dtype, bits, chunk_blocks=8, sample_symbols=1000)
    assert orc.parse_header(s_local)["n_chunks"] == 5
    s_global = _roundtrip(orc, dtype, bits, global_table=True)
    hd = orc.parse_header(s_global)
    assert hd["flags"] == 1 and hd["n_chunks"] == 1 and hd["CB"] == 37
    for B in (32, 1024, 2048, 8192, 16384):
        _roundtrip(orc, dtype, bits, block_symbols=B)


def test_ratio_large_blocks(orc):
    """C2 block sweep: a block carries 128 bytes of final lane states, so the ratio of
    W bf16 falls with B (4096 > 8192 > 16384) by about those state bytes, and stays above the
    closed-form Shannon bound."""
    n = 1 << 22
    bits = synth.normal(n, 0.02, 5, BF16)
    r = {B: len(_roundtrip(orc, BF16, bits, block_symbols=B)) / (2 * n) for B in (4096, 8192, 16384)}
    assert r[4096] > r[8192] > r[16384]
    for B in (8192, 16384):
        saved = (n // 4096 - n // B) * 128 / (2 * n)  # fewer blocks, fewer state headers
        assert abs((r[4096] - r[B]) - saved) < 0.002, (B, r)
    H = _entropy(_normal_symbol_probs(0.02))
    assert r[16384] >= (RES_BITS[BF16] + H) / (8 * EB[BF16]) - 0.002


def test_adversarial_chunk_floor(orc):
    """a symbol absent from the sampled prefix appears later."""
    n = 4096 * 8
    bits = synth.constant(n, 0x3F80, BF16)
    bits[-100:] = synth.random_bits(100, 3, BF16)
    _roundtrip(orc, BF16, bits, sample_symbols=4096)


# ----------------------------------------------------------------------------- ratios
def _entropy(p):
    p = np.asarray([x for x in p if x > 0], np.float64)
    p = p / p.sum()
    return float(-(p * np.log2(p)).sum())


def _uniform_symbol_probs(dtype):
    """|v| ~ U[0,1]: binade k (k <= -1) has mass 2^k; the top half-ulp of every
    binade rounds up into the next one (mass 2^k * 2^-(m+2)), m = fraction bits."""
    mbits = {BF16: 7, F16: 10, F32: 23}[dtype]
    probs = {}
    for k in range(-1, -150, -1):
        mass = 2.0 ** k * (1 - 2.0 ** -(mbits + 2))
        if mass < 1e-30:
            break
        probs[k] = mass
    probs[0] = probs.get(0, 0.0) + 2.0 ** -(mbits + 2)
    if dtype == F16:
        # f16 symbol = sign | 5 exponent bits | 2 fraction MSBs: the sign is 1 bit,
        # the 2 MSBs are uniform inside a binade (|v| uniform), binades below
        # 2^-14 share the subnormal code 0 and split by their own MSBs.
        return [m for m in probs.values()], 1.0 + 2.0
    return [m for m in probs.values()], 0.0


def _normal_symbol_probs(sigma):
    probs = []
    for k in range(-140, 10):
        lo, hi = 2.0 ** k, 2.0 ** (k + 1)
        probs.append(math.erf(hi / (sigma * math.sqrt(2))) - math.erf(lo / (sigma * math.sqrt(2))))
    return probs


def _bounds(n, dtype, H, B=4096, chunks=1):
    nb = n // B
    lower = (RES_BITS[dtype] + H) / (8 * EB[dtype])
    over = (0.0935 * n + nb * (128 + 16 + 4) * 8 + (64 + chunks * 520) * 8) / (8 * EB[dtype] * n)
    return lower, lower + over


@pytest.mark.parametrize("dtype,paper,tol", [(BF16, 0.64, 0.03), (F16, 0.83, 0.05), (F32, 0.82, 0.05)])
def test_ratio_uniform_vs_closed_form_and_paper(orc, dtype, paper, tol):
    """P:548-550 bf16 ~0.64; P:722 f16 0.83 / f32 0.82 (SPEC S:565-566 tolerances)."""
    n = (1 << 22) if dtype != BF16 else (1 << 24)
    bits = synth.uniform(n, 42, dtype)
    s = orc.compress(dtype, bits)
    ratio = len(s) / (n * EB[dtype])
    probs, extra = _uniform_symbol_probs(dtype)
    H = _entropy(probs) + extra
    lo, hi = _bounds(n, dtype, H, chunks=orc.parse_header(s)["n_chunks"])
    assert lo - 0.002 <= ratio <= hi + 0.002, (lo, ratio, hi)
    assert abs(ratio - paper) <= tol
    # SPEC S:566 empirical entropy oracle: within 3% absolute
    sym, _ = orc.split(dtype, bits)
    cnt = np.bincount(sym, minlength=256).astype(np.float64)
    emp = (RES_BITS[dtype] * n + (-(cnt[cnt > 0] * np.log2(cnt[cnt > 0] / n))).sum()) / (8 * EB[dtype] * n)
    assert emp <= ratio <= emp + 0.03


@pytest.mark.parametrize("kind,dtype,paper", [("W", BF16, 0.675), ("G", F32, 0.848)])
def test_ratio_normal_vs_closed_form_and_table1(orc, kind, dtype, paper):
    """Table 1: weight bf16 0.675, gradient fp32 0.848 (+-0.03)."""
    n = 1 << 22
    sigma = 0.02 if kind == "W" else 1e-3
    bits = synth.normal(n, sigma, 5, dtype)
    s = orc.compress(dtype, bits)
    ratio = len(s) / (n * EB[dtype])
    H = _entropy(_normal_symbol_probs(sigma))
    lo, hi = _bounds(n, dtype, H, chunks=orc.parse_header(s)["n_chunks"])
    assert lo - 0.002 <= ratio <= hi + 0.002, (lo, ratio, hi)
    assert abs(ratio - paper) <= 0.03


def test_ratio_activations_table1(orc):
    bits = synth.activations(1024, 3)        # [1024, 4096] bf16, 8 MiB
    ratio = len(orc.compress(BF16, bits)) / (bits.size * 2)
    assert abs(ratio - 0.679) <= 0.03        # Table 1 activation


def test_localized_vs_global_penalty(orc):
    """P:369 ~4.5% penalty on real data; local <= 1.06 x global."""
    n = 1 << 23
    bits = synth.normal(n, 0.02, 11)
    r_local = len(orc.compress(BF16, bits))
    r_global = len(orc.compress(BF16, bits, global_table=True))
    assert r_local <= 1.06 * r_global
    # stacked layers of different scales, one per 8 MiB table chunk: local
    # tables follow the drift the global table averages over
    bits2 = np.concatenate([synth.normal(1 << 22, 0.02 * 4 ** i, i) for i in range(4)])
    assert len(orc.compress(BF16, bits2)) <= 1.06 * len(orc.compress(BF16, bits2, global_table=True))


@pytest.mark.parametrize("dtype", [BF16, F16, F32])
def test_incompressible_bound(orc, dtype):
    """R13: random bits -> every block stored raw; ratio <= 1 + 2/B + 260/(B*CB) + 32/n-ish."""
    n = 4096 * 64
    bits = synth.random_bits(n, 1, dtype)
    s = orc.compress(dtype, bits)
    sec = orc.sections(s)
    d = np.frombuffer(s[sec["off_dir"]:sec["off_dir"] + 4 * 64], "<u4")
    assert np.all(d == orc.RAW_BLOCK)
    assert len(s) <= n * EB[dtype] * (1 + 4.0 / (4096 * EB[dtype])) + 64 + 520 + 16
    assert len(s) == orc.compress_bound(n, dtype)


def test_constant_tensor_ratio(orc):
    """all-1.0 bf16 -> ratio ~ 0.50 + overhead."""
    n = 1 << 20
    s = orc.compress(BF16, synth.constant(n, 0x3F80))
    assert 0.5 < len(s) / (2 * n) < 0.5 + 0.02


# ----------------------------------------------------------------------------- errors
def test_errors_and_corruption(orc):
    n = 4096 * 6 + 3
    bits = synth.normal(n, 0.02, 2)
    s = orc.compress(BF16, bits)
    assert orc.decompress(s, n + 1, BF16)[0] == orc.ERR_SIZE_MISMATCH
    assert orc.decompress(s, n, F16)[0] == orc.ERR_SIZE_MISMATCH
    assert orc.decompress(s[:-1], n, BF16)[0] == orc.ERR_CORRUPT_STREAM
    assert orc.decompress(s[:40], n, BF16)[0] == orc.ERR_CORRUPT_STREAM
    bad = bytearray(s); bad[0] ^= 1
    assert orc.decompress(bytes(bad), n, BF16)[0] == orc.ERR_CORRUPT_STREAM
    sec = orc.sections(s)
    bad = bytearray(s); bad[sec["off_tab"] + 2 * 0x7E] ^= 1            # table no longer sums to M
    assert orc.decompress(bytes(bad), n, BF16)[0] == orc.ERR_CORRUPT_STREAM
    bad = bytearray(s); bad[sec["off_dir"]] ^= 1                          # directory vs payload
    assert orc.decompress(bytes(bad), n, BF16)[0] == orc.ERR_CORRUPT_STREAM
    # random bit flips: error, or (residual/tail flips) a different output -- never a crash
    rng = np.random.default_rng(0)
    for _ in range(300):
        bad = bytearray(s)
        pos = int(rng.integers(0, len(s)))
        bad[pos] ^= 1 << int(rng.integers(0, 8))
        st, out = orc.decompress(bytes(bad), n, BF16)
        assert st in (orc.OK, orc.ERR_CORRUPT_STREAM, orc.ERR_SIZE_MISMATCH)
        if pos < 64 and st == orc.OK:          # a header flip must never pass silently with wrong data
            assert np.array_equal(out, bits)
