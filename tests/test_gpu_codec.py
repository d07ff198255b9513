"""GPU parity of the codec kernels against the CPU oracle, through the C ABI.

Bit-exact: GPU stream bytes == oracle stream bytes, GPU decode == input bytes,
across dtypes x sizes (empty, ragged, several tiles and chunks) x value
distributions x stream parameters; BASELINE C1 (4 MiB bf16 W) in full; the
1 GiB C2 shard (the bench launch configuration) by exact round trip plus
sampled tables and blocks recomputed one by one by the oracle; corrupt-stream
behaviour."""
import json
import os

import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
BF16, F16, F32, E4M3, E5M2 = 0, 1, 2, 3, 4
TD = {BF16: torch.bfloat16, F16: torch.float16, F32: torch.float32, E4M3: torch.float8_e4m3fn,
      E5M2: torch.float8_e5m2}
VIEW = {BF16: torch.int16, F16: torch.int16, F32: torch.int32, E4M3: torch.uint8, E5M2: torch.uint8}
NPV = {BF16: np.int16, F16: np.int16, F32: np.int32, E4M3: np.uint8, E5M2: np.uint8}
NPU = {BF16: np.uint16, F16: np.uint16, F32: np.uint32, E4M3: np.uint8, E5M2: np.uint8}


@pytest.fixture(scope="module")
def uz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_17172_b200 as uz
    uz.build()
    return uz


def to_dev(bits: np.ndarray, dtype: int) -> torch.Tensor:
    t = torch.from_numpy(np.ascontiguousarray(bits).view(NPV[dtype]).copy())
    return t.view(TD[dtype]).cuda()


def to_bits(t: torch.Tensor, dtype: int) -> np.ndarray:
    return t.view(VIEW[dtype]).cpu().numpy().view(NPU[dtype])


def gpu_compress(uz, bits, dtype, **params) -> bytes:
    x = to_dev(bits, dtype) if bits.size else torch.empty(0, dtype=TD[dtype], device="cuda")
    out, nbytes = uz.compress(x, **params)
    torch.cuda.synchronize()
    return out[: int(nbytes.item())].cpu().numpy().tobytes()


def gpu_decompress(uz, stream: bytes, n, dtype, in_bytes=None):
    buf = torch.from_numpy(np.frombuffer(stream, np.uint8).copy()).cuda() if stream else \
        torch.zeros(16, dtype=torch.uint8, device="cuda")
    out, st = uz.decompress(buf, n, dtype, in_bytes=in_bytes)
    torch.cuda.synchronize()
    return int(st.item()), (to_bits(out, dtype) if n else np.zeros(0))


GENS = {
    "W": lambda n, s, d: synth.normal(n, 0.02, s, d),
    "U": lambda n, s, d: synth.uniform(n, s, d),
    "special": lambda n, s, d: synth.special_mix(n, s, d),
    "random": lambda n, s, d: synth.random_bits(n, s, d),
    "zeros": lambda n, s, d: synth.constant(n, 0, d),
}


@pytest.mark.parametrize("dtype", [BF16, F16, F32])
@pytest.mark.parametrize("n", [0, 1, 4095, 4096, 4097, 3 * 4096 + 17, 40 * 4096 + 5])
@pytest.mark.parametrize("dist", list(GENS))
def test_stream_bytes_equal_oracle(uz, orc, dtype, n, dist):
    bits = GENS[dist](n, 1000 + n, dtype)
    ref = orc.compress(dtype, bits)
    got = gpu_compress(uz, bits, dtype)
    assert len(got) == len(ref)
    assert got == ref
    st, back = gpu_decompress(uz, got, n, dtype)
    assert st == 0 and np.array_equal(back, bits)


@pytest.mark.parametrize("dtype", [BF16, F16, F32])
@pytest.mark.parametrize("params", [dict(block_symbols=1024), dict(block_symbols=2048),
                                    dict(global_table=True), dict(chunk_blocks=8, sample_symbols=1000),
                                    dict(chunk_blocks=16, sample_symbols=70001, block_symbols=1024),
                                    dict(global_table=True, block_symbols=1024)])
def test_stream_params_equal_oracle(uz, orc, dtype, params):
    n = 37 * 4096 + 11
    bits = synth.normal(n, 0.02, 7, dtype)
    bits[4096 * 20:4096 * 21] = synth.random_bits(4096, 8, dtype)
    ref = orc.compress(dtype, bits, **params)
    got = gpu_compress(uz, bits, dtype, **params)
    assert got == ref
    st, back = gpu_decompress(uz, got, n, dtype)
    assert st == 0 and np.array_equal(back, bits)


def test_c1_full_4mib_bf16(uz, orc):
    """BASELINE configs[0]: one 4 MiB bf16 ~N(0,0.02) tensor, full oracle parity."""
    n = 2 * 1024 * 1024
    bits = synth.weights(n, 1000)
    ref = orc.compress(BF16, bits)
    got = gpu_compress(uz, bits, BF16)
    assert got == ref
    st, back = gpu_decompress(uz, got, n, BF16)
    assert st == 0 and np.array_equal(back, bits)
    assert abs(len(got) / (2 * n) - 0.678) < 0.005


@pytest.mark.parametrize("dtype", [BF16, F32])
def test_multichunk_48mib(uz, orc, dtype):
    n = (48 << 20) // (2 if dtype == BF16 else 4) + 123
    bits = synth.normal(n, 0.02, 3, dtype)
    assert gpu_compress(uz, bits, dtype) == orc.compress(dtype, bits)


def test_golden_streams_decode(uz):
    gold = os.path.join(os.path.dirname(__file__), "golden")
    for case in json.load(open(os.path.join(gold, "manifest.json")))["cases"]:
        bits = np.load(os.path.join(gold, case["name"] + ".npy"))
        stream = open(os.path.join(gold, case["name"] + ".uzb"), "rb").read()
        st, back = gpu_decompress(uz, stream, case["n"], case["dtype"])
        assert st == 0 and np.array_equal(back, bits), case["name"]
        cb = case["params"].get("chunk_blocks", 0)
        if cb % 8 and not case["params"].get("global_table"):
            # the GPU encoder needs chunks aligned to its 8-block tiles; it rejects others
            with pytest.raises(uz.UzipError):
                gpu_compress(uz, bits, case["dtype"], **case["params"])
            continue
        assert gpu_compress(uz, bits, case["dtype"], **case["params"]) == stream, case["name"]


def test_workspace_reuse_and_repeat(uz, orc):
    bits = synth.normal(9 * 4096 + 3, 0.02, 5)
    ref = orc.compress(BF16, bits)
    for _ in range(3):
        assert gpu_compress(uz, bits, BF16) == ref
    small = synth.normal(4096 * 2, 0.02, 6)
    assert gpu_compress(uz, small, BF16) == orc.compress(BF16, small)
    assert gpu_compress(uz, bits, BF16) == ref


def test_corrupt_and_mismatch(uz, orc):
    n = 12 * 4096 + 7
    bits = synth.normal(n, 0.02, 9)
    s = gpu_compress(uz, bits, BF16)
    assert gpu_decompress(uz, s, n + 1, BF16)[0] == uz.ERR_SIZE_MISMATCH
    assert gpu_decompress(uz, s, n, F16)[0] == uz.ERR_SIZE_MISMATCH
    assert gpu_decompress(uz, s, n, BF16, in_bytes=len(s) - 16)[0] == uz.ERR_CORRUPT_STREAM
    assert gpu_decompress(uz, s[:32], n, BF16)[0] == uz.ERR_CORRUPT_STREAM
    sec = orc.sections(s)
    rng = np.random.default_rng(1)
    for trial in range(200):
        bad = bytearray(s)
        region = trial % 4
        if region == 0:
            pos = int(rng.integers(0, 64))
        elif region == 1:
            pos = int(rng.integers(sec["off_tab"], sec["off_pay"]))
        else:
            pos = int(rng.integers(sec["off_pay"], sec["off_tail"]))
        bad[pos] ^= 1 << int(rng.integers(0, 8))
        st, out = gpu_decompress(uz, bytes(bad), n, BF16)
        ost, oout = orc.decompress(bytes(bad), n, BF16)
        # the GPU decoder rejects exactly what the oracle rejects
        assert (st == 0) == (ost == 0), (pos, st, ost)
        if st == 0:
            assert np.array_equal(out, oout)
    # the status word is reset: a good stream decodes OK again
    st, back = gpu_decompress(uz, s, n, BF16)
    assert st == 0 and np.array_equal(back, bits)


def test_c2_full_size_1gib_sampled(uz, orc):
    """BASELINE configs[1] shard (1 GiB bf16 W) in the bench's launch config:
    exact on-device round trip; tables and sampled blocks recomputed by the oracle."""
    n = 512 * 1024 * 1024
    g = torch.Generator(device="cuda")
    g.manual_seed(1001)
    x = (torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    out, nbytes = uz.compress(x)
    y, st = uz.decompress(out, n, BF16)
    torch.cuda.synchronize()
    assert int(st.item()) == 0
    assert torch.equal(x.view(torch.int16), y.view(torch.int16))
    total = int(nbytes.item())
    assert abs(total / (2 * n) - 0.678) < 0.005
    stream = out[:total].cpu().numpy()
    sec = orc.sections(stream[:64].tobytes() + b"")
    nb, nc, B, CB = sec["n_blocks"], sec["n_chunks"], sec["B"], sec["CB"]
    assert (nb, nc) == (131072, 128)
    dirv = stream[sec["off_dir"]:sec["off_dir"] + 4 * nb].view("<u4")
    coff = stream[sec["off_coff"]:sec["off_coff"] + 8 * nc].view("<u8")
    sizes = np.where(dirv == orc.RAW_BLOCK, B, (128 + 2 * dirv.astype(np.int64) + 15) // 16 * 16)
    offs = np.concatenate([[0], np.cumsum(sizes)])
    assert np.array_equal(coff, offs[np.arange(nc) * CB])
    assert offs[-1] == sec["payload_bytes"]
    xb = x.view(torch.int16)
    for c in (0, 1, 63, 127):
        sample = xb[c * CB * B: c * CB * B + 131072].cpu().numpy().view(np.uint16)
        sym, _ = orc.split(BF16, sample)
        f_ref = orc.normalize(orc.histogram(sym))
        f_gpu = stream[sec["off_tab"] + 512 * c: sec["off_tab"] + 512 * (c + 1)].view("<u2")
        assert np.array_equal(f_ref, f_gpu), c
    rng = np.random.default_rng(0)
    for b in [0, 1, CB - 1, CB, nb - 1] + list(rng.integers(0, nb, 24)):
        b = int(b)
        c = b // CB
        blk = xb[b * B:(b + 1) * B].cpu().numpy().view(np.uint16)
        sym, res = orc.split(BF16, blk)
        f = stream[sec["off_tab"] + 512 * c: sec["off_tab"] + 512 * (c + 1)].view("<u2")
        states, words = orc.encode_block(sym, f)
        ref = orc.block_bytes(states, words)
        assert dirv[b] == words.size
        got = stream[sec["off_pay"] + offs[b]: sec["off_pay"] + offs[b] + sizes[b]].tobytes()
        assert got == ref, b
        assert np.array_equal(stream[sec["off_res0"] + b * B: sec["off_res0"] + (b + 1) * B], res.astype(np.uint8))


@pytest.mark.parametrize("dtype", [BF16, F16, F32])
def test_encoder_word_overflow_rare_path(uz, orc, dtype):
    """Blocks whose first-coded rounds (the high element indices, R-1 first) are
    expensive but which still compress: the coded words outrun the symbol rows
    the encoder has consumed, and the GPU encoder takes its rare path (words
    stored straight to their final place).  Bytes must still equal the oracle."""
    B = 4096
    nb = 12
    bits = synth.constant(nb * B + 3, 0x3F80 if dtype == BF16 else (0x3C00 if dtype == F16 else 0x3F800000),
                          dtype).copy()
    rnd = synth.random_bits(nb * B, 77, dtype)
    for blk in range(nb):
        hi = 96 + 2 * blk  # rounds >= hi are random, the rest constant
        sl = slice(blk * B + hi * 32, (blk + 1) * B)
        bits[sl] = rnd[sl]
    ref = orc.compress(dtype, bits)
    got = gpu_compress(uz, bits, dtype)
    assert got == ref
    st, back = gpu_decompress(uz, got, bits.size, dtype)
    assert st == 0 and np.array_equal(back, bits)



@pytest.mark.parametrize("dtype", [BF16, F16, F32])
def test_large_coded_blocks_decoded_in_place(uz, orc, dtype):
    """Blocks that compress only a little (exponent symbols uniform over 128 values, ~7.1 bits
    each): their coded size (~3.7 KB of 4 KB) exceeds the decoder's 3200-byte smem staging area,
    so k_decode reads them in place from global memory.  Stream == oracle, round trip exact."""
    B, nb = 4096, 10
    bits = synth.random_bits(nb * B + 5, 91, dtype).copy()
    top = {BF16: 1 << 14, F16: 1 << 15, F32: 1 << 30}[dtype]  # the symbol's most significant bit
    bits &= ~np.array(top, dtype=bits.dtype)
    ref = orc.compress(dtype, bits)
    raw = bits.size * bits.itemsize
    # coded, not stored raw: between residual + 3200 B and residual + B per block
    res = {BF16: 0.5, F16: 0.5, F32: 0.75}[dtype]
    assert res + 3200 / (B * bits.itemsize) < len(ref) / raw < res + 1 / bits.itemsize - 0.005
    got = gpu_compress(uz, bits, dtype)
    assert got == ref
    st, back = gpu_decompress(uz, got, bits.size, dtype)
    assert st == 0 and np.array_equal(back, bits)


FP8_GENS = {
    "U": lambda n, s, d: synth.uniform(n, s, d),
    "W": lambda n, s, d: synth.normal(n, 0.02, s, d),
    "special": lambda n, s, d: synth.special_mix(n, s, d),
    "random": lambda n, s, d: synth.random_bits(n, s, d),
}


@pytest.mark.parametrize("dtype", [E4M3, E5M2])
@pytest.mark.parametrize("n", [0, 1, 2, 4095, 8191, 8192, 8193, 3 * 8192 + 7, 80 * 4096 + 3])
@pytest.mark.parametrize("dist", list(FP8_GENS))
def test_fp8_stream_bytes_equal_oracle(uz, orc, dtype, n, dist):
    """fp8 codecs (R23 e4m3 pairs, R24 e5m2 bytes): GPU stream == oracle stream."""
    bits = FP8_GENS[dist](n, 3000 + n, dtype)
    ref = orc.compress(dtype, bits)
    got = gpu_compress(uz, bits, dtype)
    assert got == ref
    st, back = gpu_decompress(uz, got, n, dtype)
    assert st == 0 and np.array_equal(back, bits)


@pytest.mark.parametrize("dtype", [E4M3, E5M2])
@pytest.mark.parametrize("params", [dict(block_symbols=1024), dict(global_table=True),
                                    dict(chunk_blocks=8, sample_symbols=5000, block_symbols=2048)])
def test_fp8_stream_params_equal_oracle(uz, orc, dtype, params):
    n = 45 * 4096 + 11
    bits = synth.normal(n, 0.02, 9, dtype)
    bits[4096 * 10:4096 * 12] = synth.random_bits(8192, 10, dtype)
    assert gpu_compress(uz, bits, dtype, **params) == orc.compress(dtype, bits, **params)


def test_fp8_multichunk_48mib(uz, orc):
    for dtype in (E4M3, E5M2):
        n = (48 << 20) + 123
        bits = synth.normal(n, 0.02, 4, dtype)
        assert gpu_compress(uz, bits, dtype) == orc.compress(dtype, bits)


@pytest.mark.parametrize("kind", ["tie", "coded"])
def test_stored_raw_tie_equals_oracle(uz, orc, kind):
    """The constructed tie block (roundup16(128 + 2K) == B, stored raw) and the block one 16-byte
    step below it (coded): GPU stream == oracle stream (tests/test_oracle_rawtie.py pins the oracle)."""
    from test_oracle_rawtie import tie_input
    bits = tie_input(kind)
    ref = orc.compress(BF16, bits)
    got = gpu_compress(uz, bits, BF16)
    assert got == ref
    st, back = gpu_decompress(uz, got, bits.size, BF16)
    assert st == 0 and np.array_equal(back, bits)


@pytest.mark.parametrize("dtype", [BF16, F16, F32])
@pytest.mark.parametrize("n", [3, 4096, 3 * 4096 + 17, 41 * 4096 + 5])
@pytest.mark.parametrize("B", [1024, 4096])
def test_staged_pipeline_equals_oracle_global(uz, orc, dtype, n, B):
    """Ablation baseline (f3): the staged Steps 1-3 pipeline writes the oracle's
    global-table stream byte for byte -- also with the residual plane redirected to a side buffer
    and moved into the stream afterwards (the copy-engine split-send variant)."""
    bits = synth.normal(n, 0.02, 300 + n, dtype)
    if n > 4096 * 8:
        bits[4096 * 2:4096 * 3] = synth.random_bits(4096, 9, dtype)  # stored-raw blocks too
    ref = orc.compress(dtype, bits, global_table=True, block_symbols=B)
    x = torch.from_numpy(bits.view(NPV[dtype]).copy()).view(TD[dtype]).cuda()
    out, nb = uz.compress_staged(x, block_symbols=B)
    torch.cuda.synchronize()
    assert out[: int(nb.item())].cpu().numpy().tobytes() == ref
    # copy-engine variant: residual plane to a side buffer, moved after Step 1 on a second stream
    side = torch.empty(len(ref), dtype=torch.uint8, device="cuda")
    ev = torch.cuda.Event()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    out2 = torch.zeros_like(out)
    with torch.cuda.stream(s1):
        _, nb2 = uz.compress_staged(x, out=out2, stream=s1, res_out=side, split_done=ev, block_symbols=B)
    res_bytes = orc.sections(ref)["off_tab"] - 64
    with torch.cuda.stream(s2):
        s2.wait_event(ev)
        out2[64:64 + res_bytes].copy_(side[:res_bytes], non_blocking=True)
    torch.cuda.synchronize()
    got = out2[: int(nb2.item())].cpu().numpy()
    got[64 + res_bytes:orc.sections(ref)["off_tab"]] = 0  # alignment pad after the plane (none for whole blocks)
    assert got.tobytes() == ref


def test_nvls_multicast_primitive(uz):
    """f1 building block: a one-device NVLS multicast object -- multimem.st through the multicast
    mapping lands in the bound memory (checked through the unicast mapping).  Skips when the GPU /
    driver reports no multicast support (the fan-out then stays unicast)."""
    if not uz.nvls_supported(0):
        pytest.skip("no multicast support on this device")
    st = uz.nvls_selftest(0, 8 << 20)
    if st == uz.ERR_NOT_IMPLEMENTED:
        pytest.skip("cuMulticastCreate refused on this node (single visible GPU / no multicast team)")
    assert st == 0


@pytest.mark.parametrize("dtype", [BF16, F16, F32, E4M3, E5M2])
@pytest.mark.parametrize("B", [8192, 16384])
def test_large_blocks_equal_oracle(uz, orc, dtype, B):
    """Blocks of 8192 / 16384 symbols (the C2 block sweep): several tiles, several table
    chunks (chunk_blocks=8), a stored-raw block and a ragged tail; stream bytes == oracle's, exact
    round trip.  Coded blocks this large exceed the decoder's smem staging, so they are decoded in
    place from global memory (the rare path of the 4096-symbol format)."""
    per = 2 if dtype == E4M3 else 1  # elements per symbol
    n = per * (20 * B + 11)
    bits = synth.normal(n, 0.02, 31 + B, dtype)
    bits[per * B * 9:per * B * 10] = synth.random_bits(per * B, 5, dtype)
    for params in (dict(block_symbols=B), dict(block_symbols=B, chunk_blocks=8)):
        ref = orc.compress(dtype, bits, **params)
        got = gpu_compress(uz, bits, dtype, **params)
        assert got == ref, params
        st, back = gpu_decompress(uz, got, n, dtype)
        assert st == 0 and np.array_equal(back, bits)


def test_unsupported_block_sizes_rejected(uz):
    x = torch.zeros(1 << 16, dtype=torch.bfloat16, device="cuda")
    for B in (512, 3072, 32768):
        with pytest.raises(uz.UzipError):
            uz.compress(x, block_symbols=B)


@pytest.mark.parametrize("B", [4096, 16384])
@pytest.mark.parametrize("dist", ["W", "zeros"])
def test_garbage_block_states_fail_cleanly(uz, orc, B, dist):
    """Garbage final lane states make the decoder consume words it does not have (its word index runs
    below 0; zeros give tiny, smem-staged blocks, W at 16384 large ones decoded in place): k_decode must
    report a corrupt stream, never fault, and the context stays usable."""
    n = 12 * B + 5
    bits = GENS[dist](n, 77, BF16)
    good = gpu_compress(uz, bits, BF16, block_symbols=B)
    off_pay = orc.sections(good)["off_pay"]
    rng = np.random.default_rng(B)
    for _ in range(3):  # block 0 starts the payload: overwrite its 32 final states with random words
        bad = bytearray(good)
        bad[off_pay:off_pay + 128] = rng.integers(0, 256, 128, dtype=np.uint8).tobytes()
        st, _ = gpu_decompress(uz, bytes(bad), n, BF16)
        assert st != 0
    st, back = gpu_decompress(uz, good, n, BF16)
    assert st == 0 and np.array_equal(back, bits)


def test_pair_staging_boundary_mixed_blocks(uz, orc):
    """k_decode pairs two coded bf16 blocks per warp when both fit its 1488-byte staging areas; a pair
    with an oversized block falls back to one chain per block.  Blocks here code to 1472-1744 bytes
    (W blocks next to blocks with 15 % U[-1,1] elements, one shared chunk table), so pairs of both kinds
    and a lone last block (65 blocks) occur.  Stream == oracle, round trip exact."""
    B, nb = 4096, 65
    bits = synth.normal(nb * B, 0.02, 501)
    u = synth.uniform(nb * B, 502)
    rng = np.random.default_rng(7)
    for i in np.nonzero(rng.random(nb) < 0.5)[0]:
        m = rng.random(B) < 0.15
        blk = bits[i * B:(i + 1) * B]
        blk[m] = u[i * B:(i + 1) * B][m]
    ref = orc.compress(BF16, bits)
    sec = orc.sections(ref)
    k = np.frombuffer(ref[sec["off_dir"]:sec["off_dir"] + 4 * nb], dtype=np.uint32).astype(np.int64)
    size = (128 + 2 * k + 15) // 16 * 16
    assert (size <= 1488).sum() >= 4 and (size > 1488).sum() >= 4 and size.max() < B
    got = gpu_compress(uz, bits, BF16)
    assert got == ref
    st, back = gpu_decompress(uz, got, bits.size, BF16)
    assert st == 0 and np.array_equal(back, bits)
