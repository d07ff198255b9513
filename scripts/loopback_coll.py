"""Loopback timing of the fused collectives on one GPU (N ranks share the SMs): context numbers for
tuning the receive path (table builds, tile order), not a bench line.

    python scripts/loopback_coll.py [--n 4] [--mib 256]
"""
import argparse
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4)
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--ctas_per_sm", type=int, default=1, help="total CTAs = 148 x this, split over the ranks")
    args = ap.parse_args()
    import torch
    import paper_2604_17172_b200 as uz
    uz.build()
    N = args.n
    comms = uz.Comm.init_all(N, [0] * N, max_ctas=148 * args.ctas_per_sm // N, staging_bytes=1 << 30)
    streams = [torch.cuda.Stream() for _ in range(N)]
    numel = (args.mib << 20) // 2
    g = torch.Generator(device="cuda")
    xs = []
    for r in range(N):
        g.manual_seed(100 + r)
        xs.append((torch.randn(numel, device="cuda", generator=g) * 0.02).to(torch.bfloat16))
    res = {}

    def run(name, fn):
        def step():
            ev = torch.cuda.Event()
            ev.record()
            th = []
            for r in range(N):
                streams[r].wait_event(ev)
                th.append(threading.Thread(target=fn, args=(r,)))
            for t in th:
                t.start()
            for t in th:
                t.join()
            for r in range(N):
                torch.cuda.current_stream().wait_stream(streams[r])
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.steps):
            step()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        errs = [c.async_error() for c in comms]
        res[name] = {"ms": round(ms, 3), "user_GBps": round(2 * numel / (ms / 1e3) / 1e9, 1), "errors": errs}
        print(name, res[name], flush=True)

    outs = [torch.empty(numel // N, dtype=torch.bfloat16, device="cuda") for _ in range(N)]
    run("reduce_scatter", lambda r: comms[r].reduce_scatter(outs[r], xs[r], streams[r]))
    ar = [torch.empty_like(x) for x in xs]
    run("allreduce", lambda r: comms[r].all_reduce(ar[r], xs[r], streams[r]))
    shard = [x[: numel // N] for x in xs]
    ag = [torch.empty(numel, dtype=torch.bfloat16, device="cuda") for _ in range(N)]
    run("allgather", lambda r: comms[r].all_gather(ag[r], shard[r], streams[r]))
    print(json.dumps(res))
    for c in comms:
        c.destroy()


if __name__ == "__main__":
    main()
