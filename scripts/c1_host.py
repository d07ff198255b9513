"""C1 (4 MiB bf16) host issue cost vs device time per uzip_compress / uzip_decompress call."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2604_17172_b200 as uz
n = 2 << 20
x = (torch.randn(n, device="cuda") * 0.02).to(torch.bfloat16)
buf = torch.empty(uz.compress_bound(n, uz.BF16), dtype=torch.uint8, device="cuda")
nb = torch.zeros(1, dtype=torch.int64, device="cuda")
y = torch.empty_like(x)
st = torch.zeros(1, dtype=torch.int32, device="cuda")
s = torch.cuda.Stream()
ws = uz.Workspace(0).get(uz.workspace_bytes(n, uz.BF16), s)
for _ in range(20):
    uz.compress(x, out=buf, out_bytes=nb, stream=s, ws=ws)
torch.cuda.synchronize()
for name, fn in (("compress", lambda: uz.compress(x, out=buf, out_bytes=nb, stream=s, ws=ws)),
                 ("decompress", lambda: uz.decompress(buf, n, uz.BF16, out=y, status=st, stream=s, ws=ws))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    # gate the stream so every launch is queued before the GPU starts: device time only
    gate = torch.cuda.Event()
    t0 = time.perf_counter()
    e0.record(s)
    for _ in range(200):
        fn()
    e1.record(s)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(name, "host_issue_us", round((t1 - t0) * 1e6 / 200, 2), "stream_us", round(e0.elapsed_time(e1) * 1e3 / 200, 2))
