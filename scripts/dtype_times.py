"""Per-dtype encode / decode device times (ms per 256 MiB of U[-1,1], the paper's synthetic input) of
the codec through the C ABI -- the split of bench.py's per_dtype_uniform round trips.

    python scripts/dtype_times.py [label]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_17172_b200 as uz  # noqa: E402


def main():
    label = sys.argv[1] if len(sys.argv) > 1 else "default"
    nbytes = 256 << 20
    g = torch.Generator(device="cuda")
    res = {}
    for name, tdt in (("bf16", torch.bfloat16), ("f16", torch.float16), ("f32", torch.float32),
                      ("e4m3", torch.float8_e4m3fn), ("e5m2", torch.float8_e5m2)):
        g.manual_seed(7)
        n = nbytes // torch.tensor([], dtype=tdt).element_size()
        x = (torch.rand(n, device="cuda", generator=g) * 2 - 1).to(tdt)
        dt = uz.uz_dtype(tdt)
        buf = torch.empty(uz.compress_bound(n, dt), dtype=torch.uint8, device="cuda")
        nb = torch.zeros(1, dtype=torch.int64, device="cuda")
        y = torch.empty_like(x)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        ws = uz.Workspace(0).get(uz.workspace_bytes(n, dt))
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        te = td = 0.0
        for it in range(7):
            ev[0].record()
            uz.compress(x, out=buf, out_bytes=nb, ws=ws)
            ev[1].record()
            uz.decompress(buf, n, dt, out=y, status=st, ws=ws)
            ev[2].record()
            torch.cuda.synchronize()
            if it >= 2:
                te += ev[0].elapsed_time(ev[1]) / 5
                td += ev[1].elapsed_time(ev[2]) / 5
        assert int(st.item()) == 0 and torch.equal(x.view(torch.uint8), y.view(torch.uint8))
        res[name] = (round(int(nb.item()) / nbytes, 4), round(te, 4), round(td, 4))
    print(label, res)


if __name__ == "__main__":
    main()
