"""Pin of the stored-raw rule's tie (SURVEY 8(c) O7 / DESIGN R13): a block whose coded size
roundup16(128 + 2K) equals B exactly is stored raw ("ties go to raw"); one 16-byte step below is
coded.  The two blocks are constructed (symbols uniform over A values, seeded) so that K lands in
the tie window [B/2 - 71, B/2 - 64] resp. one step below; K comes from the pinned block coder."""
import numpy as np

import oracle as _o

B = 4096
CASES = {"tie": (217, 6, 1977), "coded": (214, 19, 1970)}  # (alphabet, seed, expected K)


def tie_input(kind: str) -> np.ndarray:
    """bf16 bits of one block whose exponent symbols give the K of CASES[kind] (+ a 5-element tail)."""
    A, seed, _ = CASES[kind]
    rng = np.random.default_rng(seed * 1000 + A)
    sym = rng.integers(0, A, B).astype(np.uint16)
    res = np.random.default_rng(77).integers(0, 256, B + 5).astype(np.uint16)
    bits = ((res[:B] & 0x80) << 8) | (sym << 7) | (res[:B] & 0x7F)
    return np.concatenate([bits, res[B:] | 0x3F00]).astype(np.uint16)


def test_tie_block_is_stored_raw_and_one_step_below_is_coded(orc):
    for kind, (A, seed, K) in CASES.items():
        bits = tie_input(kind)
        sym, _ = orc.split(orc.BF16, bits[:B])
        freq = orc.normalize(np.bincount(sym, minlength=256))
        _, words = orc.encode_block(sym, freq)
        assert words.size == K
        size = (128 + 2 * K + 15) // 16 * 16
        assert size == (B if kind == "tie" else B - 16)
        stream = orc.compress(orc.BF16, bits)
        sec = orc.sections(stream)
        d = int(np.frombuffer(stream[sec["off_dir"]:sec["off_dir"] + 4], "<u4")[0])
        if kind == "tie":
            assert d == orc.RAW_BLOCK and sec["payload_bytes"] == B
        else:
            assert d == K and sec["payload_bytes"] == B - 16
        st, back = orc.decompress(stream, bits.size, orc.BF16)
        assert st == 0 and np.array_equal(back, bits)
