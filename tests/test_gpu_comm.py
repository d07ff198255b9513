"""GPU parity of the fused communication path against the CPU oracle, through the C ABI.

Several ranks run on ONE GPU (uzip_comm_init_all with repeated devices; each
rank has its own stream and a bounded CTA count so all ranks' persistent
kernels are co-resident).  The kernels, flags, credits and staging layout are
the same ones the multi-process NVLink path uses; only the peer pointers differ
(direct instead of CUDA-IPC-mapped).

Bit-exact checks (0 ulp): P2P recv == send; allgather == concatenation;
reduce-scatter / allreduce == the oracle's fixed-order fp32 fold (R11);
the UZB1 stream that lands in the receiver's staging == oracle.compress of the
round's input (wire-stream parity); compression on vs off
gives identical outputs; multi-round messages (bounded staging,
credits) and sub-threshold raw paths; NaN/Inf/denormal/-0 inputs.
"""
import numpy as np
import pytest
import torch

import synth

pytestmark = pytest.mark.gpu
BF16, F16, F32, E4M3, E5M2 = 0, 1, 2, 3, 4
TD = {BF16: torch.bfloat16, F16: torch.float16, F32: torch.float32, E4M3: torch.float8_e4m3fn,
      E5M2: torch.float8_e5m2}
VIEW = {BF16: torch.int16, F16: torch.int16, F32: torch.int32, E4M3: torch.uint8, E5M2: torch.uint8}
NPU = {BF16: np.uint16, F16: np.uint16, F32: np.uint32, E4M3: np.uint8, E5M2: np.uint8}
NPV = {BF16: np.int16, F16: np.int16, F32: np.int32, E4M3: np.uint8, E5M2: np.uint8}


@pytest.fixture(scope="module")
def uz():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_17172_b200 as uz
    uz.build()
    return uz


def dev(bits, dtype):
    t = torch.from_numpy(np.ascontiguousarray(bits).view(NPV[dtype]).copy())
    return t.view(TD[dtype]).cuda()


def host(t, dtype):
    return t.view(VIEW[dtype]).cpu().numpy().view(NPU[dtype])


def gen(dist, n, seed, dtype):
    if dist == "W":
        return synth.normal(n, 0.02, seed, dtype)
    if dist == "special":
        return synth.special_mix(n, seed, dtype)
    if dist == "U":
        return synth.uniform(n, seed, dtype)
    raise ValueError(dist)


class Group:
    """N loopback ranks on cuda:0, one stream each."""

    def __init__(self, uz, n, **cfg):
        cfg.setdefault("max_ctas", max(8, 96 // n))
        cfg.setdefault("poll_timeout_ms", 8000)
        self.comms = uz.Comm.init_all(n, **cfg)
        self.streams = [torch.cuda.Stream() for _ in range(n)]
        self.n = n

    def run(self, fn):
        torch.cuda.synchronize()
        for r, c in enumerate(self.comms):
            with torch.cuda.stream(self.streams[r]):
                fn(r, c, self.streams[r])
        torch.cuda.synchronize()
        errs = [c.async_error() for c in self.comms]
        assert errs == [0] * self.n, errs

    def close(self):
        for c in self.comms:
            c.destroy()


CFG_SMALL = dict(staging_bytes=8 << 20, min_compress_bytes=1)  # 4 MiB slots: multi-round messages


@pytest.mark.parametrize("dtype", [BF16, F16, F32])
@pytest.mark.parametrize("n", [1, 4095, 3 * 4096 + 17, 300 * 1024 + 5, 3 * (1 << 20) + 77])
def test_p2p_bit_exact(uz, dtype, n):
    g = Group(uz, 2, **CFG_SMALL)
    try:
        bits = gen("W", n, 11 + n, dtype)
        x = dev(bits, dtype)
        y = torch.full_like(x, 7)

        def step(r, c, s):
            if r == 0:
                c.send(x, 1, s)
            else:
                c.recv(y, 0, s)
        g.run(step)
        assert np.array_equal(host(y, dtype), bits)
        st = g.comms[0].stats()
        assert st["compressed"] and st["raw_bytes"] == n * (4 if dtype == F32 else 2)
    finally:
        g.close()


def test_p2p_wire_stream_equals_oracle(uz, orc):
    """The bytes that land in the receiver's staging are the oracle's UZB1 stream."""
    g = Group(uz, 2, staging_bytes=64 << 20, min_compress_bytes=1)
    try:
        n = 5 * (1 << 20) + 123
        bits = synth.weights(n, 5)
        x = dev(bits, BF16)
        y = torch.empty_like(x)
        g.run(lambda r, c, s: c.send(x, 1, s) if r == 0 else c.recv(y, 0, s))
        ref = orc.compress(BF16, bits)
        wire = g.comms[1].read_staging(0, 0, len(ref))
        assert wire == ref
        st = g.comms[0].stats()
        assert st["wire_bytes"] == len(ref)
        assert np.array_equal(host(y, BF16), bits)
    finally:
        g.close()


def test_p2p_many_rounds_and_credits(uz, orc):
    """A message of 7 rounds through 2 slots, repeated: exercises credit waits and epochs."""
    g = Group(uz, 2, staging_bytes=4 << 20, min_compress_bytes=1)
    try:
        n = 7 * (1 << 20) + 9
        for it in range(3):
            bits = synth.weights(n, 100 + it)
            x = dev(bits, BF16)
            y = torch.empty_like(x)
            g.run(lambda r, c, s: c.send(x, 1, s) if r == 0 else c.recv(y, 0, s))
            assert np.array_equal(host(y, BF16), bits), it
    finally:
        g.close()


@pytest.mark.parametrize("nr", [2, 3, 4])
@pytest.mark.parametrize("dtype", [BF16, F32])
@pytest.mark.parametrize("dist", ["W", "special"])
def test_allgather(uz, nr, dtype, dist):
    g = Group(uz, nr, **CFG_SMALL)
    try:
        n = 2 * (1 << 20) + 4096 * 3 + 5 if dtype == BF16 else (1 << 20) + 77
        ins = [gen(dist, n, 1000 * r + 3, dtype) for r in range(nr)]
        xs = [dev(b, dtype) for b in ins]
        outs = [torch.empty(nr * n, dtype=TD[dtype], device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.all_gather(outs[r], xs[r], s))
        ref = np.concatenate(ins)
        for r in range(nr):
            assert np.array_equal(host(outs[r], dtype), ref), r
    finally:
        g.close()


@pytest.mark.parametrize("nr", [2, 3, 4])
@pytest.mark.parametrize("dtype", [BF16, F16, F32])
def test_reduce_scatter(uz, orc, nr, dtype):
    g = Group(uz, nr, **CFG_SMALL)
    try:
        m = (1 << 20) + 4096 * 2 + 8  # per-rank shard (ragged tail, 16-byte aligned shards)
        ins = [gen("W", nr * m, 77 + r, dtype) for r in range(nr)]
        xs = [dev(b, dtype) for b in ins]
        outs = [torch.empty(m, dtype=TD[dtype], device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.reduce_scatter(outs[r], xs[r], s))
        ref = orc.reduce_scatter(dtype, ins, nr)
        for r in range(nr):
            assert np.array_equal(host(outs[r], dtype), ref[r]), r
    finally:
        g.close()


@pytest.mark.parametrize("nr", [2, 4])
@pytest.mark.parametrize("dtype", [BF16, F16, F32])
@pytest.mark.parametrize("dist", ["W", "special"])
def test_allreduce(uz, orc, nr, dtype, dist):
    g = Group(uz, nr, **CFG_SMALL)
    try:
        n = nr * ((1 << 20) + 4096 + 8)
        ins = [gen(dist, n, 500 + r, dtype) for r in range(nr)]
        xs = [dev(b, dtype) for b in ins]
        outs = [torch.empty(n, dtype=TD[dtype], device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.all_reduce(outs[r], xs[r], s))
        ref = orc.allreduce(dtype, ins)
        for r in range(nr):
            assert np.array_equal(host(outs[r], dtype), ref), r
    finally:
        g.close()


def test_allreduce_in_place_and_transparency(uz, orc):
    """In-place allreduce; compressed and uncompressed paths give identical bits."""
    nr, n = 4, 4 * (600 * 1024)
    ins = [synth.activations(n // 4096, 40 + r) for r in range(nr)]
    results = {}
    for mode, cfg in (("on", dict(min_compress_bytes=1)), ("off", dict(min_compress_bytes=(1 << 64) - 1))):
        g = Group(uz, nr, staging_bytes=16 << 20, **cfg)
        try:
            xs = [dev(b, BF16) for b in ins]
            g.run(lambda r, c, s: c.all_reduce(xs[r], None, s))
            results[mode] = [host(x, BF16) for x in xs]
            assert g.comms[0].stats()["compressed"] == (mode == "on")
        finally:
            g.close()
    ref = orc.allreduce(BF16, ins)
    for r in range(nr):
        assert np.array_equal(results["on"][r], ref)
        assert np.array_equal(results["off"][r], ref)


@pytest.mark.parametrize("op", [1, 2])  # UZIP_MIN, UZIP_MAX (R25)
@pytest.mark.parametrize("nr", [2, 3])
@pytest.mark.parametrize("dtype", [BF16, F16, F32])
@pytest.mark.parametrize("compress", [True, False])
def test_min_max_reduce_scatter_and_allreduce(uz, orc, op, nr, dtype, compress):
    """min / max folds (NaN propagates, -0 < +0) on the compressed and the raw path == oracle."""
    cfg = dict(CFG_SMALL) if compress else dict(staging_bytes=8 << 20, min_compress_bytes=(1 << 64) - 1)
    g = Group(uz, nr, **cfg)
    try:
        m = (1 << 19) + 4096 + 8
        ins = [gen("special" if r % 2 else "W", nr * m, 3100 + 7 * r + op, dtype) for r in range(nr)]
        xs = [dev(b, dtype) for b in ins]
        outs = [torch.empty(m, dtype=TD[dtype], device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.reduce_scatter(outs[r], xs[r], s, op=op))
        ref = orc.reduce_scatter(dtype, ins, nr, op)
        for r in range(nr):
            assert np.array_equal(host(outs[r], dtype), ref[r]), r
        assert g.comms[0].stats()["compressed"] == compress
        ar = [torch.empty(nr * m, dtype=TD[dtype], device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.all_reduce(ar[r], xs[r], s, op=op))
        ref = orc.allreduce(dtype, ins, op)
        for r in range(nr):
            assert np.array_equal(host(ar[r], dtype), ref), r
    finally:
        g.close()


def test_reduce_rejects_unknown_op_and_fp8(uz):
    g = Group(uz, 2, **CFG_SMALL)
    try:
        x = torch.zeros(2 * 4096, dtype=torch.bfloat16, device="cuda")
        with pytest.raises(uz.UzipError):
            g.comms[0].all_reduce(x, None, None, op=3)
        f = torch.zeros(2 * 4096, dtype=torch.float8_e4m3fn, device="cuda")
        with pytest.raises(uz.UzipError):
            g.comms[0].all_reduce(f, None, None, op=1)
    finally:
        g.close()


@pytest.mark.parametrize("pipe_mib", [16, 24])
@pytest.mark.parametrize("issue", ["send_first", "threads"])
def test_p2p_many_multichunk_rounds_no_starvation(uz, pipe_mib, issue):
    """Dozens of 2-3-chunk rounds through 2 slots with sender and receiver sharing the GPU: the
    credit for round k comes from the receiver's round k-2 of the same call.  Regression: when
    every CTA of the sender's kernel spun on that credit, the receiver's kernel could not get SM
    slots and both timed out (now k_credit waits, one thread, before the fused launch)."""
    import threading
    comms = uz.Comm.init_all(2, [0, 0], staging_bytes=1 << 30, max_ctas=296, pipe_chunk_bytes=pipe_mib << 20,
                             poll_timeout_ms=5000)
    try:
        n = 384 << 20  # 768 MiB bf16: 48 (16 MiB) or 32 (24 MiB) rounds of 2-3 table chunks
        g = torch.Generator(device="cuda")
        g.manual_seed(pipe_mib)
        x = (torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
        y = torch.empty_like(x)
        s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
        for _ in range(2):
            y.zero_()
            torch.cuda.synchronize()
            snd = lambda: comms[0].send(x, 1, s0)  # noqa: E731
            rcv = lambda: comms[1].recv(y, 0, s1)  # noqa: E731
            if issue == "send_first":
                snd()
                rcv()
            else:
                th = [threading.Thread(target=snd), threading.Thread(target=rcv)]
                for t in th:
                    t.start()
                for t in th:
                    t.join()
            torch.cuda.synchronize()
            assert [c.async_error() for c in comms] == [0, 0], [c.error_detail() for c in comms]
            assert torch.equal(x.view(torch.int16), y.view(torch.int16))
    finally:
        for c in comms:
            c.destroy()


def test_reduce_scatter_rejects_unaligned_shards(uz):
    g = Group(uz, 2, **CFG_SMALL)
    try:
        x = torch.zeros(2 * 1001, dtype=torch.bfloat16, device="cuda")
        y = torch.zeros(1001, dtype=torch.bfloat16, device="cuda")
        with pytest.raises(uz.UzipError):
            g.comms[0].reduce_scatter(y, x)
    finally:
        g.close()


@pytest.mark.parametrize("nr", [2, 3, 4])
@pytest.mark.parametrize("dtype", [BF16, F32])
@pytest.mark.parametrize("count", [1, 4095, 3 * 4096 + 1, (1 << 20) + 12345, 3 * (1 << 20) + 7])
@pytest.mark.parametrize("compress", [True, False])
def test_allreduce_any_count(uz, orc, nr, dtype, count, compress):
    """Allreduce of any element count, like NCCL (R21): N shards of ceil(count/N) elements rounded up to
    16 bytes, the last ones shorter or empty; compressed (fused one-pass rounds) and raw; multi-round
    with 4 MiB slots; bit-exact against the oracle's fixed-order fold."""
    cfg = dict(staging_bytes=8 << 20, min_compress_bytes=1 if compress else (1 << 64) - 1)
    g = Group(uz, nr, **cfg)
    try:
        ins = [gen("W", count, 7000 + 31 * r + count % 97, dtype) for r in range(nr)]
        xs = [dev(b, dtype) for b in ins]
        outs = [torch.empty(count, dtype=TD[dtype], device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.all_reduce(outs[r], xs[r], s))
        ref = orc.allreduce(dtype, ins)
        for r in range(nr):
            assert np.array_equal(host(outs[r], dtype), ref), r
    finally:
        g.close()


def test_below_threshold_raw_path(uz, orc):
    """Messages under min_compress_bytes move raw, same results."""
    nr = 2
    g = Group(uz, nr, staging_bytes=4 << 20)  # default threshold 1 MiB
    try:
        n = 2 * 1008  # < 1 MiB, 16-byte shards
        ins = [synth.weights(n, 9 + r) for r in range(nr)]
        xs = [dev(b, BF16) for b in ins]
        outs = [torch.empty(n, dtype=torch.bfloat16, device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.all_reduce(outs[r], xs[r], s))
        ref = orc.allreduce(BF16, ins)
        for r in range(nr):
            assert np.array_equal(host(outs[r], BF16), ref)
        st = g.comms[0].stats()
        assert not st["compressed"] and st["wire_bytes"] == st["raw_bytes"]
    finally:
        g.close()


def test_mixed_sequence_epochs(uz, orc):
    """P2P and collectives interleaved on the same channels keep their epochs in step."""
    nr = 3
    g = Group(uz, nr, **CFG_SMALL)
    try:
        n = (1 << 20) + 11
        a = [synth.weights(n, 900 + r) for r in range(nr)]
        xs = [dev(b, BF16) for b in a]
        ys = [torch.empty(nr * n, dtype=torch.bfloat16, device="cuda") for _ in range(nr)]
        p = torch.empty(n, dtype=torch.bfloat16, device="cuda")
        for it in range(2):
            g.run(lambda r, c, s: c.send(xs[0], 2, s) if r == 0 else (c.recv(p, 0, s) if r == 2 else None))
            assert np.array_equal(host(p, BF16), a[0])
            g.run(lambda r, c, s: c.all_gather(ys[r], xs[r], s))
            for r in range(nr):
                assert np.array_equal(host(ys[r], BF16), np.concatenate(a))
    finally:
        g.close()


@pytest.mark.parametrize("nr", [2, 3, 4])
@pytest.mark.parametrize("dtype", [BF16, F32])
@pytest.mark.parametrize("root", [0, 1])
def test_broadcast_scatter_relay(uz, orc, nr, dtype, root):
    """Broadcast (RL weight sync): compressed scatter + relay for >= 3 ranks, fan-out for 2;
    every rank ends with the root's bytes; multi-round pieces; uneven last piece."""
    g = Group(uz, nr, **CFG_SMALL)
    try:
        n = 3 * (1 << 20) + 4096 * 5 + 13 if dtype == BF16 else (1 << 20) + 4096 + 7
        bits = gen("W", n, 31 + nr, dtype)
        bufs = [dev(bits, dtype) if r == root else torch.full((n,), 3, dtype=TD[dtype], device="cuda")
                for r in range(nr)]
        for _ in range(2):
            g.run(lambda r, c, s: c.broadcast(bufs[r], root, s))
            for r in range(nr):
                assert np.array_equal(host(bufs[r], dtype), bits), r
    finally:
        g.close()


def test_broadcast_relay_wire_streams_equal_oracle(uz, orc):
    """With 3 ranks the root's piece streams, and the relayed copies, are the oracle's streams."""
    nr, root = 3, 0
    g = Group(uz, nr, staging_bytes=64 << 20, min_compress_bytes=1)
    try:
        n = 4 * (1 << 20) + 40
        bits = synth.weights(n, 77)
        bufs = [dev(bits, BF16) if r == root else torch.empty(n, dtype=torch.bfloat16, device="cuda")
                for r in range(nr)]
        g.run(lambda r, c, s: c.broadcast(bufs[r], root, s))
        P = ((n + 1) // 2 + 15) // 16 * 16  # pieces of 16 elements (comm.cu)
        pieces = [bits[:P], bits[P:]]
        refs = [orc.compress(BF16, pc) for pc in pieces]
        # piece 0 -> rank 1 from root; rank 1 relays it to rank 2 (src 1); piece 1 -> rank 2, relayed to rank 1
        assert g.comms[1].read_staging(root, 0, len(refs[0])) == refs[0]
        assert g.comms[2].read_staging(root, 0, len(refs[1])) == refs[1]
        assert g.comms[2].read_staging(1, 0, len(refs[0])) == refs[0]
        assert g.comms[1].read_staging(2, 0, len(refs[1])) == refs[1]
        for r in range(nr):
            assert np.array_equal(host(bufs[r], BF16), bits)
    finally:
        g.close()


@pytest.mark.parametrize("nr", [2, 3, 4])
@pytest.mark.parametrize("dtype", [BF16, F16, F32])
def test_alltoall(uz, nr, dtype):
    """All-to-all: out_r[i] == in_i[r] for every pair, compressed per-peer streams."""
    g = Group(uz, nr, **CFG_SMALL)
    try:
        c = (1 << 20) + 4096 + 8
        ins = [gen("W", nr * c, 600 + r, dtype) for r in range(nr)]
        xs = [dev(b, dtype) for b in ins]
        outs = [torch.empty(nr * c, dtype=TD[dtype], device="cuda") for _ in range(nr)]
        for _ in range(2):
            g.run(lambda r, cm, s: cm.all_to_all(outs[r], xs[r], s))
            for r in range(nr):
                ref = np.concatenate([ins[i][r * c:(r + 1) * c] for i in range(nr)])
                assert np.array_equal(host(outs[r], dtype), ref), r
    finally:
        g.close()


def test_missing_peer_times_out_instead_of_hanging(uz):
    """Failure detection: a recv whose sender never comes raises UZIP_ERR_TIMEOUT in the
    communicator's async error word after poll_timeout_ms; the kernel exits, the GPU stays usable."""
    import time
    g = Group(uz, 2, staging_bytes=4 << 20, min_compress_bytes=1, poll_timeout_ms=300)
    try:
        y = torch.empty(1 << 20, dtype=torch.bfloat16, device="cuda")
        t0 = time.time()
        g.comms[1].recv(y, 0, g.streams[1])
        torch.cuda.synchronize()
        assert time.time() - t0 < 30
        assert g.comms[1].async_error() == uz.ERR_TIMEOUT
        # the device is fine: a plain codec call still works
        x = torch.randn(4096 * 3, device="cuda").to(torch.bfloat16)
        out, nb = uz.compress(x)
        back, st = uz.decompress(out, x.numel(), uz.BF16)
        torch.cuda.synchronize()
        assert int(st.item()) == 0 and torch.equal(back.view(torch.int16), x.view(torch.int16))
    finally:
        g.close()


@pytest.mark.parametrize("max_ctas", [296, 1000])
def test_p2p_large_full_occupancy(uz, max_ctas):
    """The bench's loopback configuration: large multi-round message, both ranks' persistent kernels
    as wide as the GPU allows (sender and receiver compete for SMs)."""
    g = Group(uz, 2, staging_bytes=256 << 20, max_ctas=max_ctas, poll_timeout_ms=5000)
    try:
        n = 192 << 20  # 384 MiB bf16: several rounds through 128 MiB slots
        gg = torch.Generator(device="cuda")
        gg.manual_seed(5)
        x = (torch.randn(n, device="cuda", generator=gg) * 0.02).to(torch.bfloat16)
        y = torch.empty_like(x)
        for _ in range(3):
            y.fill_(0)
            torch.cuda.synchronize()
            g.comms[0].send(x, 1, g.streams[0])
            g.comms[1].recv(y, 0, g.streams[1])
            torch.cuda.synchronize()
            errs = [c.async_error() for c in g.comms]
            if errs != [0, 0]:
                print("ERROR_DETAIL", [c.error_detail() for c in g.comms], flush=True)
            assert errs == [0, 0]
            assert torch.equal(x.view(torch.int16), y.view(torch.int16))
    finally:
        g.close()



@pytest.mark.parametrize("dtype", [E4M3, E5M2])
def test_fp8_p2p_allgather_alltoall_broadcast(uz, orc, dtype):
    """fp8 on the communication path (R22): P2P (with the wire stream == oracle), allgather with
    ragged counts, all-to-all and the relayed broadcast are bit-exact; reductions are rejected."""
    nr = 3
    g = Group(uz, nr, staging_bytes=32 << 20, min_compress_bytes=1)
    try:
        n = 3 * (1 << 20) + 4096 * 2 + 5
        bits = gen("W", n, 70, dtype)
        x = dev(bits, dtype)
        y = torch.empty_like(x)
        g.run(lambda r, c, s: c.send(x, 1, s) if r == 0 else (c.recv(y, 0, s) if r == 1 else None))
        assert np.array_equal(host(y, dtype), bits)
        ref = orc.compress(dtype, bits)
        assert g.comms[1].read_staging(0, 0, len(ref)) == ref
        m = (1 << 20) + 4096 + 3
        ins = [gen("U", m, 80 + r, dtype) for r in range(nr)]
        xs = [dev(b, dtype) for b in ins]
        outs = [torch.empty(nr * m, dtype=TD[dtype], device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.all_gather(outs[r], xs[r], s))
        for r in range(nr):
            assert np.array_equal(host(outs[r], dtype), np.concatenate(ins))
        cc = (1 << 20) + 32
        a2a_in = [gen("W", nr * cc, 90 + r, dtype) for r in range(nr)]
        a2a_x = [dev(b, dtype) for b in a2a_in]
        a2a_o = [torch.empty(nr * cc, dtype=TD[dtype], device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.all_to_all(a2a_o[r], a2a_x[r], s))
        for r in range(nr):
            assert np.array_equal(host(a2a_o[r], dtype),
                                  np.concatenate([a2a_in[i][r * cc:(r + 1) * cc] for i in range(nr)]))
        bufs = [dev(bits, dtype) if r == 0 else torch.empty(n, dtype=TD[dtype], device="cuda") for r in range(nr)]
        g.run(lambda r, c, s: c.broadcast(bufs[r], 0, s))
        for r in range(nr):
            assert np.array_equal(host(bufs[r], dtype), bits)
        with pytest.raises(uz.UzipError):
            g.comms[0].all_reduce(xs[0][: 3 * 4096])
    finally:
        g.close()


@pytest.mark.parametrize("codec", [dict(block_symbols=1024), dict(block_symbols=2048, chunk_blocks=16),
                                   dict(global_table=True)])
def test_collectives_with_codec_params(uz, orc, codec):
    """The wire format's parameters (block size, chunk size, global table) flow through the
    communicator: P2P wire stream == oracle stream with the same params; allreduce bit-exact."""
    nr = 2
    g = Group(uz, nr, staging_bytes=64 << 20, min_compress_bytes=1, **codec)
    try:
        n = 3 * (1 << 20) + 4096 * 7 + 11
        bits = synth.weights(n, 123)
        x = dev(bits, BF16)
        y = torch.empty_like(x)
        g.run(lambda r, c, s: c.send(x, 1, s) if r == 0 else c.recv(y, 0, s))
        assert np.array_equal(host(y, BF16), bits)
        ref = orc.compress(BF16, bits, **codec)
        assert g.comms[1].read_staging(0, 0, len(ref)) == ref
        m = nr * ((1 << 20) + 4096 * 3 + 8)
        ins = [synth.activations(m // 4096, 300 + r)[:m] if m % 4096 == 0 else synth.weights(m, 300 + r)
               for r in range(nr)]
        xs = [dev(b, BF16) for b in ins]
        outs = [torch.empty(m, dtype=torch.bfloat16, device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.all_reduce(outs[r], xs[r], s))
        refar = orc.allreduce(BF16, ins)
        for r in range(nr):
            assert np.array_equal(host(outs[r], BF16), refar)
    finally:
        g.close()


def _act(n, seed, dtype):
    """Activation-like values (N(0,1) x per-channel exp(N(0, 0.5^2)) scale, two outlier
    channels x 64), generated on the GPU so the full BASELINE sizes stay fast."""
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    h = 4096
    scale = torch.exp(torch.randn(h, device="cuda", generator=g) * 0.5)
    scale[7] *= 64
    scale[1337] *= 64
    return (torch.randn(n // h, h, device="cuda", generator=g) * scale).reshape(-1).to(TD[dtype])


@pytest.mark.parametrize("dtype", [BF16])
def test_full_size_allreduce_reduce_scatter_n8_sampled(uz, orc, dtype):
    """BASELINE configs[3] at its largest point: 8 ranks (loopback on one GPU), 256 MiB bf16 activation
    allreduce and reduce-scatter.  Every rank's allreduce output is bitwise identical, and 8192 sampled
    elements equal the oracle's fixed-order fp32 fold of the 8 inputs (R11); reduce-scatter shards are
    checked the same way."""
    nr, n = 8, (256 << 20) // 2
    g = Group(uz, nr, max_ctas=148 * 3 // nr, poll_timeout_ms=20000)
    try:
        xs = [_act(n, 4000 + r, dtype) for r in range(nr)]
        outs = [torch.empty_like(x) for x in xs]
        g.run(lambda r, c, s: c.all_reduce(outs[r], xs[r], s))
        for r in range(1, nr):
            assert torch.equal(outs[r].view(VIEW[dtype]), outs[0].view(VIEW[dtype]))
        idx = np.sort(np.random.default_rng(5).choice(n, 8192, replace=False))
        it = torch.from_numpy(idx).cuda()
        ins = [host(x[it], dtype) for x in xs]
        assert np.array_equal(host(outs[0][it], dtype), orc.reduce(dtype, ins))
        m = n // nr
        shards = [torch.empty(m, dtype=TD[dtype], device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.reduce_scatter(shards[r], xs[r], s))
        for r in range(nr):
            j = np.sort(np.random.default_rng(10 + r).choice(m, 1024, replace=False))
            jt = torch.from_numpy(j + r * m).cuda()
            ref = orc.reduce(dtype, [host(x[jt], dtype) for x in xs])
            assert np.array_equal(host(shards[r][torch.from_numpy(j).cuda()], dtype), ref)
    finally:
        g.close()


def test_full_size_allgather_4gib_n8(uz):
    """BASELINE configs[4] at its largest point: 4 GiB allgather output over 8 ranks (512 MiB bf16
    weights per rank), every rank's output == the concatenation of the inputs, compared in full."""
    nr, n = 8, (512 << 20) // 2
    g = Group(uz, nr, max_ctas=148 * 3 // nr, poll_timeout_ms=20000)
    try:
        xs = []
        for r in range(nr):
            gg = torch.Generator(device="cuda")
            gg.manual_seed(5000 + r)
            xs.append((torch.randn(n, device="cuda", generator=gg) * 0.02).to(torch.bfloat16))
        cat = torch.cat(xs).view(torch.int16)
        outs = [torch.empty(nr * n, dtype=torch.bfloat16, device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.all_gather(outs[r], xs[r], s))
        for r in range(nr):
            assert torch.equal(outs[r].view(torch.int16), cat)
        del outs, cat
    finally:
        g.close()
        torch.cuda.empty_cache()


def qwen25_7b_shapes():
    """Qwen2.5-7B-shaped weight tensors: 28 layers x {q [3584,3584] + bias, k/v
    [512,3584] + bias, o [3584,3584], gate/up [18944,3584], down [3584,18944], 2 norms [3584]} +
    embed and lm_head [152064,3584] + final norm = 339 tensors, 7,615,616,512 elements."""
    h, kv, ff, vocab = 3584, 512, 18944, 152064
    layer = [(h, h), (h,), (kv, h), (kv,), (kv, h), (kv,), (h, h), (ff, h), (ff, h), (h, ff), (h,), (h,)]
    return [(vocab, h)] + layer * 28 + [(h,), (vocab, h)]


def test_full_size_rl_weight_sync_n8(uz):
    """BASELINE configs[2] in full: every tensor of a Qwen2.5-7B-shaped bf16 model (~15.2 GB, W recipe,
    own seed per tensor) broadcast from rank 0 to ranks 1-7 (loopback on one GPU), one call per
    tensor (the sub-1 MiB biases and norms take the raw path); every receiver's bytes == the root's."""
    shapes = qwen25_7b_shapes()
    assert len(shapes) == 339 and sum(int(np.prod(s)) for s in shapes) == 7_615_616_512
    nr = 8
    g = Group(uz, nr, max_ctas=148 * 3 // nr, poll_timeout_ms=20000)
    try:
        big = max(int(np.prod(s)) for s in shapes)
        bufs = [torch.empty(big, dtype=torch.bfloat16, device="cuda") for _ in range(nr)]
        gg = torch.Generator(device="cuda")
        for i, s in enumerate(shapes):
            n = int(np.prod(s))
            gg.manual_seed(7000 + i)
            bufs[0][:n].copy_(torch.randn(n, device="cuda", generator=gg) * 0.02)
            for r in range(1, nr):
                bufs[r][:n].fill_(7)
            g.run(lambda r, c, st: c.broadcast(bufs[r][:n], 0, st))
            ref = bufs[0][:n].view(torch.int16)
            for r in range(1, nr):
                assert torch.equal(bufs[r][:n].view(torch.int16), ref), (i, s, r)
    finally:
        g.close()
        torch.cuda.empty_cache()


@pytest.mark.parametrize("mode", ["one_message", "per_layer"])
def test_full_size_kv_cache_p2p(uz, mode):
    """BASELINE configs[4] KV-cache transfer in full: Llama-3-8B vLLM KV blocks for 7680 tokens
    (480 blocks x 32 layers x 64 KiB = 960 MiB bf16; K = N(0,1) x per-dim exp(N(0, 0.5^2)), V = N(0,1)),
    sent GPU "0" -> "1" (loopback) as one message or as 32 per-layer messages of 30 MiB; recv == send."""
    g = Group(uz, 2, max_ctas=296, poll_timeout_ms=20000)
    try:
        gg = torch.Generator(device="cuda")
        gg.manual_seed(8000)
        layers, nb = 32, 480
        kscale = torch.exp(torch.randn(layers, 1, 1, 8, 128, device="cuda", generator=gg) * 0.5)
        k = torch.randn(layers, nb, 16, 8, 128, device="cuda", generator=gg) * kscale
        v = torch.randn(layers, nb, 16, 8, 128, device="cuda", generator=gg)
        x = torch.stack([k, v], dim=2).to(torch.bfloat16).contiguous()  # [layer, block, K/V, 16, 8, 128]
        del k, v
        assert x.numel() * 2 == 960 << 20
        y = torch.zeros_like(x)
        if mode == "one_message":
            g.run(lambda r, c, s: c.send(x.view(-1), 1, s) if r == 0 else c.recv(y.view(-1), 0, s))
        else:
            def per_layer(r, c, s):
                for l in range(layers):
                    if r == 0:
                        c.send(x[l].view(-1), 1, s)
                    else:
                        c.recv(y[l].view(-1), 0, s)
            g.run(per_layer)
        assert torch.equal(y.view(torch.int16), x.view(torch.int16))
        st = g.comms[0].stats()
        assert 0.5 < st["wire_bytes"] / st["raw_bytes"] < 0.85, st  # compressed (activation-like ratio)
    finally:
        g.close()
        torch.cuda.empty_cache()


def test_back_to_back_collectives_rank_major_issue(uz, orc):
    """A queue of collectives issued without synchronisation, rank by rank (rank 0 enqueues its whole
    sequence before rank 1 enqueues anything): allreduce / allgather / reduce-scatter of 2-32 MiB,
    several rounds through 8 MiB slots, so producers of later calls owe credits to consumers that are
    still queued.  Allgather compared in full; allreduce / reduce-scatter on sampled elements vs the
    oracle's fixed-order fold."""
    nr = 4
    g = Group(uz, nr, staging_bytes=16 << 20, max_ctas=148 * 3 // nr, poll_timeout_ms=20000)
    try:
        ops = [("ar", 15 << 20), ("ag", 4 << 20), ("rs", 12 << 20), ("ar", 1 << 20), ("ag", 8 << 20),
               ("ar", 8 << 20), ("rs", 2 << 20), ("ar", 16 << 20)]  # element counts (bf16)
        data, outs = [], []
        for k, (op, n) in enumerate(ops):
            xs = [_act(n, 9000 + 10 * k + r, BF16) for r in range(nr)]
            data.append(xs)
            m = {"ar": n, "ag": n * nr, "rs": n // nr}[op]
            outs.append([torch.empty(m, dtype=torch.bfloat16, device="cuda") for _ in range(nr)])
        torch.cuda.synchronize()
        for r, c in enumerate(g.comms):  # rank-major issue, no synchronisation in between
            s = g.streams[r]
            with torch.cuda.stream(s):
                for k, (op, n) in enumerate(ops):
                    if op == "ar":
                        c.all_reduce(outs[k][r], data[k][r], s)
                    elif op == "ag":
                        c.all_gather(outs[k][r], data[k][r], s)
                    else:
                        c.reduce_scatter(outs[k][r], data[k][r], s)
        torch.cuda.synchronize()
        assert [c.async_error() for c in g.comms] == [0] * nr
        rng = np.random.default_rng(17)
        for k, (op, n) in enumerate(ops):
            xs, ys = data[k], outs[k]
            if op == "ag":
                cat = torch.cat(xs).view(torch.int16)
                for r in range(nr):
                    assert torch.equal(ys[r].view(torch.int16), cat), (k, r)
            elif op == "ar":
                for r in range(1, nr):
                    assert torch.equal(ys[r].view(torch.int16), ys[0].view(torch.int16)), (k, r)
                it = torch.from_numpy(np.sort(rng.choice(n, 2048, replace=False))).cuda()
                ref = orc.reduce(BF16, [host(x[it], BF16) for x in xs])
                assert np.array_equal(host(ys[0][it], BF16), ref), k
            else:
                m = n // nr
                for r in range(nr):
                    j = np.sort(rng.choice(m, 512, replace=False))
                    ref = orc.reduce(BF16, [host(x[torch.from_numpy(j + r * m).cuda()], BF16) for x in xs])
                    assert np.array_equal(host(ys[r][torch.from_numpy(j).cuda()], BF16), ref), (k, r)
    finally:
        g.close()


@pytest.mark.parametrize("chunk_blocks", [0, 8])
def test_p2p_decode_runs(uz, chunk_blocks):
    """A ~1 GiB message in one round (16384+ tiles): the receiver takes its tiles in runs of 8 (one
    decode-table build per run); with 8-block chunks every tile of a run has its own table, and the
    last run is ragged.  recv == send, both sides' kernels sized for the whole GPU in turn."""
    g = Group(uz, 2, staging_bytes=3 << 30, max_ctas=296, poll_timeout_ms=20000,
              **({"chunk_blocks": chunk_blocks} if chunk_blocks else {}))
    try:
        n = (1 << 29) + 3 * 4096 * 8 + 4096 + 5  # ragged: a partial last tile and a raw tail
        gg = torch.Generator(device="cuda")
        gg.manual_seed(77)
        x = (torch.randn(n, device="cuda", generator=gg) * 0.02).to(torch.bfloat16)
        y = torch.zeros_like(x)
        g.run(lambda r, c, s: c.send(x, 1, s) if r == 0 else c.recv(y, 0, s))
        assert torch.equal(y.view(torch.int16), x.view(torch.int16))
    finally:
        g.close()
        torch.cuda.empty_cache()


@pytest.mark.parametrize("nr", [2, 3])
@pytest.mark.parametrize("dtype", [BF16, F16, F32])
@pytest.mark.parametrize("codec", [dict(), dict(block_symbols=1024, chunk_blocks=16), dict(block_symbols=2048)])
def test_allreduce_fused_wire_streams_equal_oracle(uz, orc, nr, dtype, codec):
    """One-pass allreduce (a9, R26): every stream on the wire is the oracle's.  Reduce-scatter
    phase: shard r of rank s's input, default sampling; allgather phase: rank s's REDUCED shard,
    coded in the same launch as the reduction with each chunk's table sampled from its first tile
    (sample_symbols = 8 B).  Outputs bit-exact against the fixed-order fold."""
    g = Group(uz, nr, staging_bytes=64 << 20, min_compress_bytes=1, **codec)
    try:
        m = (1 << 20) + 4096 * 5 + 8 if dtype != F32 else (1 << 19) + 4096 * 3 + 4
        ins = [gen("W", nr * m, 900 + 13 * r + dtype, dtype) for r in range(nr)]
        xs = [dev(b, dtype) for b in ins]
        outs = [torch.empty(nr * m, dtype=TD[dtype], device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.all_reduce(outs[r], xs[r], s))
        ref = orc.allreduce(dtype, ins)
        for r in range(nr):
            assert np.array_equal(host(outs[r], dtype), ref), r
        for s, d, phase, blob in orc.wire_streams("allreduce", dtype, ins, **codec):
            slot = 0 if phase == "rs" else 1  # the launch uses both slots of every pair
            assert g.comms[d].read_staging(s, slot, len(blob)) == blob, (phase, s, d)
        st = g.comms[0].stats()
        assert st["compressed"] and st["wire_bytes"] < st["raw_bytes"]
    finally:
        g.close()


@pytest.mark.parametrize("dist", ["W", "special"])
def test_allreduce_fused_many_rounds_and_chunks(uz, orc, dist):
    """The one-pass allreduce over many rounds (2 MiB slots: both slots of every pair are used by
    each launch, so every round waits for the previous round's credits) and many table chunks per
    round (chunk_blocks=8: every tile publishes its own table); incompressible (special) data
    exercises stored-raw blocks of the re-encoded shard."""
    nr = 3
    g = Group(uz, nr, staging_bytes=4 << 20, min_compress_bytes=1, chunk_blocks=8)
    try:
        m = 3 * (1 << 20) + 4096 * 3 + 16
        ins = [gen(dist, nr * m, 4400 + r, BF16) for r in range(nr)]
        xs = [dev(b, BF16) for b in ins]
        for it in range(2):
            outs = [torch.empty(nr * m, dtype=torch.bfloat16, device="cuda") for _ in range(nr)]
            g.run(lambda r, c, s: c.all_reduce(outs[r], xs[r], s))
            ref = orc.allreduce(BF16, ins)
            for r in range(nr):
                assert np.array_equal(host(outs[r], BF16), ref), (it, r)
    finally:
        g.close()


@pytest.mark.parametrize("kind", ["allgather", "reduce_scatter"])
@pytest.mark.parametrize("nr", [2, 3, 4])
def test_collective_wire_streams_equal_oracle(uz, orc, kind, nr):
    """Every (src, dst) stream of a compressed allgather / reduce-scatter that lands in dst's
    staging is the oracle's O13 stream (oracle.wire_streams), byte for byte."""
    g = Group(uz, nr, staging_bytes=64 << 20, min_compress_bytes=1)
    try:
        m = (1 << 20) + 4096 * 9 + 8
        if kind == "allgather":
            ins = [synth.weights(m, 61 + r) for r in range(nr)]
            xs = [dev(b, BF16) for b in ins]
            outs = [torch.empty(nr * m, dtype=torch.bfloat16, device="cuda") for _ in range(nr)]
            g.run(lambda r, c, s: c.all_gather(outs[r], xs[r], s))
        else:
            ins = [synth.weights(nr * m, 81 + r) for r in range(nr)]
            xs = [dev(b, BF16) for b in ins]
            outs = [torch.empty(m, dtype=torch.bfloat16, device="cuda") for _ in range(nr)]
            g.run(lambda r, c, s: c.reduce_scatter(outs[r], xs[r], s))
        for s, d, _, blob in orc.wire_streams(kind, BF16, ins):
            assert g.comms[d].read_staging(s, 0, len(blob)) == blob, (s, d)
    finally:
        g.close()


@pytest.mark.parametrize("B", [8192, 16384])
def test_large_blocks_p2p_allgather(uz, orc, B):
    """Blocks of 8192 / 16384 symbols through the communicator (C2 block sweep): the P2P wire stream
    == the oracle's with the same params, allgather bit-exact; reductions reject B > 4096."""
    nr = 2
    g = Group(uz, nr, staging_bytes=64 << 20, min_compress_bytes=1, block_symbols=B)
    try:
        n = 3 * (1 << 20) + B * 7 + 11
        bits = synth.weights(n, 77 + B)
        x = dev(bits, BF16)
        y = torch.empty_like(x)
        g.run(lambda r, c, s: c.send(x, 1, s) if r == 0 else c.recv(y, 0, s))
        assert np.array_equal(host(y, BF16), bits)
        ref = orc.compress(BF16, bits, block_symbols=B)
        assert g.comms[1].read_staging(0, 0, len(ref)) == ref
        m = (1 << 20) + 3 * B + 5
        ins = [synth.weights(m, 500 + r) for r in range(nr)]
        xs = [dev(b, BF16) for b in ins]
        outs = [torch.empty(nr * m, dtype=torch.bfloat16, device="cuda") for _ in range(nr)]
        g.run(lambda r, c, s: c.all_gather(outs[r], xs[r], s))
        for r in range(nr):
            assert np.array_equal(host(outs[r], BF16), np.concatenate(ins))
        with pytest.raises(uz.UzipError):
            g.comms[0].all_reduce(outs[0], outs[0])
    finally:
        g.close()


@pytest.mark.parametrize("dtype", [BF16, F16, F32])
@pytest.mark.parametrize("codec", [dict(), dict(chunk_blocks=16)])
def test_paired_tile_receiver_small(uz, orc, dtype, codec):
    """Decode-only receivers pair consecutive tiles of a run (two rANS chains per warp).  Runs only
    form on >= 128 MiB rounds by default, so UZIP_DEC_RUN (read once per process: see
    test_paired_tile_receiver_forced_runs) forces them; here: whatever the run length, a message with
    incompressible blocks, several chunks and a ragged tail arrives bit-exact with the oracle's stream."""
    g = Group(uz, 2, staging_bytes=64 << 20, min_compress_bytes=1, **codec)
    try:
        n = 41 * 8 * 4096 + 4096 * 3 + 7
        bits = gen("W", n, 606 + dtype, dtype)
        bits[4096 * 50:4096 * 53] = synth.random_bits(4096 * 3, 9, dtype)  # stored-raw blocks
        x = dev(bits, dtype)
        y = torch.empty_like(x)
        g.run(lambda r, c, s: c.send(x, 1, s) if r == 0 else c.recv(y, 0, s))
        assert np.array_equal(host(y, dtype), bits)
        ref = orc.compress(dtype, bits, **codec)
        assert g.comms[1].read_staging(0, 0, len(ref)) == ref
    finally:
        g.close()
