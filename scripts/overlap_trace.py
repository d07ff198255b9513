"""Overlap evidence from the library's tile trace (UZIP_TRACE=1): no timeline profiler needed.

    UZIP_TRACE=1 python scripts/overlap_trace.py [--mib 256] [--out profiles/r02_overlap_trace.json]

Two loopback ranks on one GPU (both ranks' kernels share it, so absolute times are a lower bound; the
receiver is launched first -- a receiver launched after its sender does not get SMs on the shared GPU
until the sender's persistent kernel is done, RECV_FIRST=0 shows that case):
  * split-send P2P: per tile, the sender's flag release (E) and the receiver's decode (D); reports the
    fraction of the receiver's tiles decoded before the sender released its last tile (transfer and
    decode overlapping the encode) and the median flag-to-decoded latency per tile;
  * one-pass allreduce (a9): allgather-stream tiles released while later tiles of the same rank's shard
    are still being reduced -- each reduced tile leaves at once, no phase barrier.
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    os.environ.setdefault("UZIP_TRACE", "1")
    import numpy as np
    import torch
    import paper_2604_17172_b200 as uz
    n = (args.mib << 20) // 2
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    x = (torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    y = torch.empty_like(x)
    comms = uz.Comm.init_all(2, [0, 0], max_ctas=296, staging_bytes=1 << 30)
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):  # warm-up, then one traced call
        comms[0].trace(), comms[1].trace()
        if os.environ.get("RECV_FIRST", "1") == "1":  # the receiver holds its SM share before the sender starts
            comms[1].recv(y, 0, s1)
            comms[0].send(x, 1, s0)
        else:
            comms[0].send(x, 1, s0)
            comms[1].recv(y, 0, s1)
        torch.cuda.synchronize()
    assert torch.equal(x.view(torch.int16), y.view(torch.int16))
    te, td = comms[0].trace(), comms[1].trace()
    flag = te[te[:, 0] == 2]
    done = td[td[:, 0] == 4]
    last_flag = flag[:, 3].max()
    t0 = min(te[te[:, 0] == 1][:, 3].min(), done[:, 3].min())
    fl = dict(zip(flag[:, 2], flag[:, 3]))
    lat = [d - fl[t] for t, d in zip(done[:, 2], done[:, 3]) if t in fl]
    res = {"workload": f"loopback split-send P2P of {args.mib} MiB bf16 W, 2 ranks on one B200",
           "tiles": int(len(flag)),
           "receiver_tiles_done_before_sender_finished": round(float((done[:, 3] < last_flag).mean()), 4),
           "sender_span_us": round((last_flag - t0) / 1e3, 1),
           "receiver_last_done_after_sender_last_flag_us": round((done[:, 3].max() - last_flag) / 1e3, 1),
           "median_flag_to_decoded_us": round(float(np.median(lat)) / 1e3, 1)}
    # one-pass allreduce: allgather-stream tiles released while reduce-scatter tiles still go out
    a = [x.clone(), (x * 2).to(torch.bfloat16)]
    o = [torch.empty_like(a[0]), torch.empty_like(a[1])]
    comms[0].trace(), comms[1].trace()
    s = [s0, s1]
    for r in range(2):
        with torch.cuda.stream(s[r]):
            comms[r].all_reduce(o[r], a[r], s[r])
    torch.cuda.synchronize()
    tr = comms[0].trace()
    fl = tr[tr[:, 0] == 2]
    ag = fl[fl[:, 1] == 1]  # E job 1: the allgather stream of the reduced shard (job 0: reduce-scatter)
    red = tr[(tr[:, 0] == 4) & (tr[:, 1] == 0)]  # D job 0: the reduce items (decode + fold + re-encode)
    if len(red) and len(ag):
        res["allreduce_one_pass"] = {
            "reduced_tiles": int(len(red)), "ag_tiles": int(len(ag)),
            "first_ag_flag_before_last_reduce_us": round((red[:, 3].max() - ag[:, 3].min()) / 1e3, 1),
            "ag_tiles_released_before_last_reduced_tile": round(float((ag[:, 3] < red[:, 3].max()).mean()), 4)}
    for c in comms:
        c.destroy()
    print(json.dumps(res))
    if args.out:
        open(args.out, "w").write(json.dumps(res, indent=1) + "\n")


if __name__ == "__main__":
    main()
