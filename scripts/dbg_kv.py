"""Debug: per-layer KV P2P on loopback ranks (32 x 30 MiB), both issue orders; prints error detail."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17172_b200 as uz

order = sys.argv[1] if len(sys.argv) > 1 else "sends_first"
nmsg = int(sys.argv[2]) if len(sys.argv) > 2 else 32
mib = int(sys.argv[3]) if len(sys.argv) > 3 else 30
ctas = int(sys.argv[4]) if len(sys.argv) > 4 else 296
uz.build()
comms = uz.Comm.init_all(2, [0, 0], max_ctas=ctas, poll_timeout_ms=5000)
ss = [torch.cuda.Stream() for _ in range(2)]
n = (mib << 20) // 2
x = (torch.randn(nmsg, n, device="cuda") * 0.02).to(torch.bfloat16)
y = torch.zeros_like(x)
torch.cuda.synchronize()
if order == "sends_first":
    for l in range(nmsg):
        comms[0].send(x[l], 1, ss[0])
    for l in range(nmsg):
        comms[1].recv(y[l], 0, ss[1])
else:
    for l in range(nmsg):
        comms[0].send(x[l], 1, ss[0])
        comms[1].recv(y[l], 0, ss[1])
torch.cuda.synchronize()
errs = [c.async_error() for c in comms]
print(order, nmsg, mib, ctas, "errs", errs, "detail", [c.error_detail() for c in comms] if any(errs) else "",
      "equal", torch.equal(x.view(torch.int16), y.view(torch.int16)), flush=True)
