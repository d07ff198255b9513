"""Pins of the oracle's O13 wire-stream enumeration (oracle.wire_streams), CPU only.

What is pinned: each stream decodes to exactly the bytes the collective's plain definition moves
(P2P recv == send, shard j of in_r for reduce-scatter, the fixed-order fold R of
shard j for the allreduce's allgather phase); the stream count and routing match the one-step /
two-step exchanges of SURVEY 8(e); the allreduce's allgather-phase header records the R26 sample
(8 B symbols) and its ratio stays within S:567's 1.06 x of the default sampled table.
"""
import numpy as np
import pytest

import synth


@pytest.mark.parametrize("N", [2, 3, 4])
@pytest.mark.parametrize("dtype", [0, 1, 2])
def test_allreduce_streams_decode_to_the_plain_definition(orc, N, dtype):
    m = 3 * 4096 * 8 + 4096 + 5 if dtype != 2 else 2 * 4096 * 8 + 7
    ins = [synth.normal(N * m, 0.02, 70 + r, dtype) for r in range(N)]
    ws = orc.wire_streams("allreduce", dtype, ins)
    rs = [w for w in ws if w[2] == "rs"]
    ag = [w for w in ws if w[2] == "ag"]
    assert len(rs) == N * (N - 1) and len(ag) == N * (N - 1)
    assert sorted((s, d) for s, d, _, _ in rs) == sorted((s, d) for s in range(N) for d in range(N) if d != s)
    red = orc.allreduce(dtype, ins)
    # the fold is the plain definition: numpy float32 sequential sum for bf16 (exact widening)
    for s, d, _, blob in rs:
        st, bits = orc.decompress(blob, m, dtype)
        assert st == 0 and np.array_equal(bits, np.asarray(ins[s]).reshape(-1)[d * m:(d + 1) * m])
    for s, d, _, blob in ag:
        st, bits = orc.decompress(blob, m, dtype)
        assert st == 0 and np.array_equal(bits, red[s * m:(s + 1) * m])
        assert orc.parse_header(blob)["S"] == 8 * 4096  # R26: one tile's symbols
    # the same blob goes to every peer of a source
    for s in range(N):
        assert len({blob for s2, _, _, blob in ag if s2 == s}) == 1


def test_r26_tile_sample_ratio_within_spec_bound(orc):
    """a localized (sampled) table costs at most 6 % of ratio vs the global table; the R26
    tile sample (32 Ki symbols) vs the default 256 KiB sample on 8 MiB chunks of W data."""
    n = 3 * (1 << 22) + 4096 * 9 + 3
    x = synth.weights(n, 9)
    glob = len(orc.compress(0, x, global_table=True))
    dflt = len(orc.compress(0, x))
    tile = len(orc.compress(0, x, sample_symbols=8 * 4096))
    assert tile <= 1.06 * glob and dflt <= 1.06 * glob
    assert abs(tile - dflt) / dflt < 0.005


def test_p2p_allgather_reduce_scatter_routing(orc):
    N, m = 3, 4096 * 9 + 1
    ins = [synth.weights(N * m, 5 + r) for r in range(N)]
    (s, d, ph, blob), = orc.wire_streams("p2p", 0, ins[:1])
    assert (s, d, ph) == (0, 1, "p2p") and orc.decompress(blob, N * m, 0)[1].tobytes() == ins[0].tobytes()
    ag = orc.wire_streams("allgather", 0, ins)
    assert len(ag) == N * (N - 1)
    for s, d, _, blob in ag:
        assert np.array_equal(orc.decompress(blob, N * m, 0)[1], ins[s])
    rs = orc.wire_streams("reduce_scatter", 0, ins)
    assert [w[:3] for w in rs] == [w[:3] for w in orc.wire_streams("allreduce", 0, ins) if w[2] == "rs"]
