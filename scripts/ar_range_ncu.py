"""DRAM bytes and duration of ONE loopback allreduce (all ranks' kernels together) for ncu range
replay, which -- unlike kernel replay -- lets the co-resident ranks' persistent kernels run side by
side:

    ncu --replay-mode app-range --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        python scripts/ar_range_ncu.py --n 2 --mib 256
"""
import argparse
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=2)
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--op", default="allreduce")
    args = ap.parse_args()
    import torch
    import paper_2604_17172_b200 as uz
    N = args.n
    comms = uz.Comm.init_all(N, [0] * N, max_ctas=148 // N, staging_bytes=1 << 30)
    streams = [torch.cuda.Stream() for _ in range(N)]
    numel = (args.mib << 20) // 2
    g = torch.Generator(device="cuda")
    xs = []
    for r in range(N):
        g.manual_seed(100 + r)
        xs.append((torch.randn(numel, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
    outs = [torch.empty_like(x) for x in xs]

    def once():
        th = [threading.Thread(target=lambda r=r: comms[r].all_reduce(outs[r], xs[r], streams[r])) for r in range(N)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        torch.cuda.synchronize()

    once()
    once()
    torch.cuda.profiler.start()
    once()
    torch.cuda.profiler.stop()
    assert [c.async_error() for c in comms] == [0] * N
    print("ok", N, args.mib, os.environ.get("UZIP_AR_FUSED", "1"))
    for c in comms:
        c.destroy()


if __name__ == "__main__":
    main()
