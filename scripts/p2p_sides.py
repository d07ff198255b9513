"""Each side of the fused split-send P2P timed alone on one B200 (loopback ranks, one round):
the sender's k_fused E items with no receiver running, then the receiver's D items on a staging slot
that is already complete -- so their speed can be compared with uzip_compress / uzip_decompress."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_17172_b200 as uz

n = (1 << 30) // 2
uz.build()
x = (torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16)
y = torch.empty_like(x)
res = {}
for ctas in (0, 296):
    comms = uz.Comm.init_all(2, [0, 0], staging_bytes=3 << 30, max_ctas=ctas, poll_timeout_ms=20000)
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    ts, tr = [], []
    for it in range(6):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        torch.cuda.synchronize()
        e[0].record(s0)
        comms[0].send(x, 1, s0)
        e[1].record(s0)
        torch.cuda.synchronize()
        e[2].record(s1)
        comms[1].recv(y, 0, s1)
        e[3].record(s1)
        torch.cuda.synchronize()
        if it >= 2:
            ts.append(e[0].elapsed_time(e[1]))
            tr.append(e[2].elapsed_time(e[3]))
    ok = torch.equal(x.view(torch.int16), y.view(torch.int16)) and [c.async_error() for c in comms] == [0, 0]
    res[f"max_ctas_{ctas}"] = {"send_ms": round(min(ts), 4), "recv_ms": round(min(tr), 4), "ok": ok}
    for c in comms:
        c.destroy()
print(json.dumps(res))
