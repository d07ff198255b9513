"""Golden UZB1 streams: committed oracle output must decode
bit-exactly and re-encode byte-identically (format stability)."""
import json
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CASES = json.load(open(os.path.join(GOLD, "manifest.json")))["cases"]


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_golden_stream_stable(orc, case):
    bits = np.load(os.path.join(GOLD, case["name"] + ".npy"))
    stream = open(os.path.join(GOLD, case["name"] + ".uzb"), "rb").read()
    assert len(stream) == case["stream_bytes"]
    st, out = orc.decompress(stream, case["n"], case["dtype"])
    assert st == orc.OK and np.array_equal(out, bits)
    assert orc.compress(case["dtype"], bits, **case["params"]) == stream
