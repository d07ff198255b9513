"""Write the golden UZB1 fixtures under tests/golden/ ("committed golden
blobs for each dtype decode bit-exactly and re-encode byte-identically").

Calls ONLY oracle/ (never the CUDA path).  Rerun after a deliberate format
change; the commit must name the DESIGN.md reading that changed.

    python scripts/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

CASES = [
    # name, dtype, generator, params
    ("bf16_w_3blk_tail", oracle.BF16, lambda: synth.weights(3 * 4096 + 17, 1000), {}),
    ("f16_u_2blk_tail", oracle.F16, lambda: synth.uniform(2 * 4096 + 5, 1001, oracle.F16), {}),
    ("f32_g_2blk_tail", oracle.F32, lambda: synth.gradients(2 * 4096 + 3, 1002), {}),
    ("bf16_special_raw", oracle.BF16, lambda: synth.special_mix(2 * 4096, 1003), {}),
    ("bf16_w_global_b1024", oracle.BF16, lambda: synth.weights(5 * 1024 + 1, 1004),
     {"global_table": True, "block_symbols": 1024}),
    ("bf16_w_chunks", oracle.BF16, lambda: synth.weights(9 * 1024, 1005),
     {"block_symbols": 1024, "chunk_blocks": 4, "sample_symbols": 2000}),
    ("bf16_w_chunks8", oracle.BF16, lambda: synth.weights(20 * 1024 + 7, 1006),
     {"block_symbols": 1024, "chunk_blocks": 8, "sample_symbols": 3000}),
    ("e4m3_u_2blk_odd", oracle.E4M3, lambda: synth.uniform(2 * 8192 + 5, 1007, oracle.E4M3), {}),
    ("e5m2_w_3blk_tail", oracle.E5M2, lambda: synth.weights(3 * 4096 + 9, 1008, oracle.E5M2), {}),
]


def main():
    import json
    out = os.path.join(ROOT, "tests", "golden")
    os.makedirs(out, exist_ok=True)
    manifest = {"source": "scripts/make_golden.py (oracle/ only)", "cite": "SPEC S:574; DESIGN.md Format",
                "cases": []}
    for name, dtype, gen, params in CASES:
        bits = gen()
        stream = oracle.compress(dtype, bits, **params)
        np.save(os.path.join(out, name + ".npy"), bits)
        with open(os.path.join(out, name + ".uzb"), "wb") as f:
            f.write(stream)
        manifest["cases"].append({"name": name, "dtype": dtype, "n": int(bits.size), "params": params,
                                  "stream_bytes": len(stream)})
        print(name, bits.size, len(stream))
    with open(os.path.join(out, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)


if __name__ == "__main__":
    main()
