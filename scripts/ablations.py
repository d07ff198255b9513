"""Ablations of the fused P2P design on one B200.

    python scripts/ablations.py [--bytes N] [--steps K] [--out FILE]

All legs move the same 1 GiB bf16 N(0, 0.02) tensor from loopback rank 0 to rank 1 (both ranks on this
one GPU, so sender and receiver share SMs and HBM -- a lower bound for the NVLink case) and check the
bytes:
  * fused           uzip_send / uzip_recv, default configuration (one persistent kernel per side per
                    256 MiB round, tile-granular overlap);
  * chunked_8MiB    the same calls with pipe_chunk_bytes = 8 MiB: one UZB1 stream and one launch per 8 MiB
                    chunk -- the paper's "8 MB chunked pipeline" / NCCL-slice granularity;
  * chunked_1MiB    the same at 1 MiB (chunked_64MiB / chunked_256MiB: the rest of BASELINE configs[1]'s
                    pipeline-chunk sweep);
  * block_<B>       the fused path with 1024- / 2048- / 8192- / 16384-symbol codec blocks (configs[1]'s
                    block-size sweep; codec_blocks: the codec alone per B);
  * encode_send     uzip_compress of the whole message, a device copy of the stream (the wire), then
                    uzip_decompress -- serial, no overlap (fig:compare_with_native_pipeline);
  * sm_limited      the fused path with each side's kernel capped at max_ctas CTAs (fig:resource_usage;
                    a CTA cap stands in for Green Contexts, f3).
Timing: CUDA events on rank 0's stream around K steps after warm-up (inputs exceed L2).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GB = 1e9


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--bytes", type=int, default=1 << 30)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    import torch
    import paper_2604_17172_b200 as uz
    uz.build()
    n = args.bytes // 2
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    x = (torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    y = torch.empty_like(x)
    raw = 2 * n
    res = {"workload": f"loopback P2P of {raw >> 20} MiB bf16 N(0,0.02) on one B200", "legs": {}}

    def timed(step, s0):
        for _ in range(args.warmup):
            step()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s0)
        for _ in range(args.steps):
            step()
        e1.record(s0)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / args.steps

    def p2p_leg(name, **cfg):
        cfg.setdefault("staging_bytes", 1 << 30)
        comms = uz.Comm.init_all(2, [0, 0], **cfg)
        s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
        y.zero_()

        threaded = "pipe_chunk_bytes" in cfg

        def step():
            s1.wait_stream(s0)
            if threaded:  # each side from its own thread, as two processes would: hundreds of small rounds
                th = [threading.Thread(target=comms[0].send, args=(x, 1, s0)),  # can fill one thread's
                      threading.Thread(target=comms[1].recv, args=(y, 0, s1))]  # launch queue first
                for t in th:
                    t.start()
                for t in th:
                    t.join()
            else:
                comms[0].send(x, 1, s0)
                comms[1].recv(y, 0, s1)
            s0.wait_stream(s1)

        ms = timed(step, s0)
        ok = torch.equal(x.view(torch.int16), y.view(torch.int16)) and [c.async_error() for c in comms] == [0, 0]
        st = comms[0].stats()
        for c in comms:
            c.destroy()
        res["legs"][name] = {"GBps": round(raw / (ms / 1e3) / GB, 2), "ms": round(ms, 4), "bit_exact": bool(ok),
                             "wire_ratio": round(st["wire_bytes"] / max(1, st["raw_bytes"]), 5),
                             "config": {k: v for k, v in cfg.items() if k != "staging_bytes"}}
        print(name, res["legs"][name], flush=True)

    p2p_leg("fused", max_ctas=2 * 148)
    p2p_leg("chunked_8MiB", max_ctas=2 * 148, pipe_chunk_bytes=8 << 20)
    p2p_leg("chunked_1MiB", max_ctas=2 * 148, pipe_chunk_bytes=1 << 20)
    for mib in (64, 256):  # BASELINE configs[1] pipeline-chunk sweep (whole slots = "fused" above)
        p2p_leg(f"chunked_{mib}MiB", max_ctas=2 * 148, pipe_chunk_bytes=mib << 20)
    for bs in (1024, 2048, 8192, 16384):  # ... and its codec block-size sweep (4096 = "fused")
        p2p_leg(f"block_{bs}", max_ctas=2 * 148, block_symbols=bs)
    for m in (16, 37, 74, 148):
        p2p_leg(f"sm_limited_{m}ctas", max_ctas=m)

    # encode-send: compress, copy the stream (the wire), decompress; serial
    stream = torch.cuda.Stream()
    cap = uz.compress_bound(n, uz.BF16)
    sbuf = torch.empty(cap, dtype=torch.uint8, device="cuda")
    rbuf = torch.empty(cap, dtype=torch.uint8, device="cuda")
    nb = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    ws = uz.Workspace(0).get(uz.workspace_bytes(n, uz.BF16), stream)
    with torch.cuda.stream(stream):
        uz.compress(x, out=sbuf, out_bytes=nb, stream=stream, ws=ws)
    torch.cuda.synchronize()
    wire = int(nb.item())
    y.zero_()

    def es_step():
        with torch.cuda.stream(stream):
            uz.compress(x, out=sbuf, out_bytes=nb, stream=stream, ws=ws)
            rbuf[:wire].copy_(sbuf[:wire])
            uz.decompress(rbuf, n, uz.BF16, out=y, status=st, stream=stream, ws=ws, in_bytes=wire)

    ms = timed(es_step, stream)
    ok = int(st.item()) == 0 and torch.equal(x.view(torch.int16), y.view(torch.int16))
    res["legs"]["encode_send"] = {"GBps": round(raw / (ms / 1e3) / GB, 2), "ms": round(ms, 4), "bit_exact": bool(ok),
                                  "wire_ratio": round(wire / raw, 5),
                                  "note": "uzip_compress + device copy of the stream + uzip_decompress, serial"}
    print("encode_send", res["legs"]["encode_send"], flush=True)
    codec_legs(uz, x, args, timed, res)
    line = json.dumps(res)
    print(line)
    if args.out:
        open(args.out, "w").write(line + "\n")


def codec_legs(uz, x, args, timed, res):
    """Compression side alone (1 GiB bf16 W, one GPU), fused vs the paper's staged pipeline:
      * fused_local / fused_global: uzip_compress with per-chunk sampled tables (default) and with one
        global table (global_table = 1);
      * staged_3pass: uzip_compress_staged -- Step 1 split + global histogram, Step 2 every block into a
        temporary slot, Step 3 scan + copy into one buffer; same stream as fused_global;
      * staged_ce_split_send: the same with the residual plane written to a side buffer and moved into
        the stream by the copy engine (cudaMemcpyAsync on a second stream after Step 1) while Steps 2-3
        run -- the split-send of P:300-311 on copy engines;
      * green_ctx_<k>sm: fused_local in a Green Context of k SMs (cuGreenCtxCreate), the paper's
        SM-limited runs (fig:resource_usage)."""
    import torch
    n = x.numel()
    raw = 2 * n
    stream = torch.cuda.Stream()
    cap = uz.compress_bound(n, uz.BF16)
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    nb = torch.zeros(1, dtype=torch.int64, device="cuda")
    legs = {}

    def leg(name, step, ref=None):
        ms = timed(step, stream)
        torch.cuda.synchronize()
        got = out[: int(nb.item())].cpu().numpy().tobytes() if ref is not None else None
        legs[name] = {"GBps_uncompressed": round(raw / (ms / 1e3) / GB, 2), "ms": round(ms, 4),
                      "ratio": round(int(nb.item()) / raw, 5)}
        if ref is not None:
            legs[name]["bytes_equal_fused_global"] = got == ref
        print(name, legs[name], flush=True)

    ws = uz.Workspace(0).get(max(uz.workspace_bytes(n, uz.BF16, global_table=True), uz.workspace_bytes(n, uz.BF16)),
                             stream)

    def fused(glob):
        def step():
            with torch.cuda.stream(stream):
                uz.compress(x, out=out, out_bytes=nb, stream=stream, ws=ws, global_table=glob)
        return step
    leg("fused_local", fused(False))
    leg("fused_global", fused(True))
    ref = out[: int(nb.item())].cpu().numpy().tobytes()
    sws = torch.zeros(uz.lib().uzip_staged_workspace_bytes(n, uz.BF16, None), dtype=torch.uint8, device="cuda")

    def staged():
        with torch.cuda.stream(stream):
            uz.compress_staged(x, out=out, out_bytes=nb, stream=stream, ws=sws)
    leg("staged_3pass", staged, ref)
    side = torch.empty(n, dtype=torch.uint8, device="cuda")
    ev = torch.cuda.Event()
    s2 = torch.cuda.Stream()

    def staged_ce():
        with torch.cuda.stream(stream):
            uz.compress_staged(x, out=out, out_bytes=nb, stream=stream, ws=sws, res_out=side, split_done=ev)
        s2.wait_event(ev)
        with torch.cuda.stream(s2):
            out[64:64 + n].copy_(side, non_blocking=True)  # the copy engine moves the residual plane
        stream.wait_stream(s2)
    leg("staged_ce_split_send", staged_ce, ref)
    res["codec_legs"] = legs
    # block-size sweep of the codec alone (configs[1]: B in {1024 ... 16384}): compress and decompress
    blk = {}
    y = torch.empty_like(x)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    for bs in (1024, 2048, 4096, 8192, 16384):
        wsb = uz.Workspace(0).get(uz.workspace_bytes(n, uz.BF16, block_symbols=bs), stream)
        if uz.compress_bound(n, uz.BF16, block_symbols=bs) > out.numel():
            out = torch.empty(uz.compress_bound(n, uz.BF16, block_symbols=bs), dtype=torch.uint8, device="cuda")

        def comp():
            with torch.cuda.stream(stream):
                uz.compress(x, out=out, out_bytes=nb, stream=stream, ws=wsb, block_symbols=bs)

        def dec():
            with torch.cuda.stream(stream):
                uz.decompress(out, n, uz.BF16, out=y, status=st, stream=stream, ws=wsb)
        mc = timed(comp, stream)
        md = timed(dec, stream)
        torch.cuda.synchronize()
        ok = int(st.item()) == 0 and torch.equal(x.view(torch.int16), y.view(torch.int16))
        blk[f"B{bs}"] = {"compress_ms": round(mc, 4), "decompress_ms": round(md, 4),
                         "ratio": round(int(nb.item()) / raw, 5), "bit_exact": ok}
        print("codec_block", bs, blk[f"B{bs}"], flush=True)
    res["codec_blocks"] = blk
    try:
        res["green_ctx"] = green_ctx_legs(uz, x, args)
    except Exception as e:  # report, do not fail the other legs
        res["green_ctx"] = {"error": repr(e)[:300]}
    print("green_ctx", res["green_ctx"], flush=True)


def green_ctx_legs(uz, x, args):
    """uzip_compress in Green Contexts holding k of the GPU's SMs (driver API through cuda-python)."""
    import torch
    from cuda.bindings import driver as d

    def ok(r):
        if not isinstance(r, tuple):
            r = (r,)
        if int(r[0]) != 0:
            raise RuntimeError(f"driver error {r[0]}")
        return None if len(r) == 1 else (r[1] if len(r) == 2 else r[1:])

    ok(d.cuInit(0))
    dev = ok(d.cuDeviceGet(0))
    sm_res = ok(d.cuDeviceGetDevResource(dev, d.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
    n = x.numel()
    raw = 2 * n
    cap = uz.compress_bound(n, uz.BF16)
    out = torch.empty(cap, dtype=torch.uint8, device="cuda")
    nb = torch.zeros(1, dtype=torch.int64, device="cuda")
    ws = uz.Workspace(0).get(uz.workspace_bytes(n, uz.BF16))
    prim = ok(d.cuCtxGetCurrent())
    res = {}
    for k in (16, 32, 64, 128):  # SMs per green context
        groups, ngroups, _rem = ok(d.cuDevSmResourceSplitByCount(1, sm_res, 0, k))
        desc = ok(d.cuDevResourceGenerateDesc([groups[0]] if isinstance(groups, list) else groups, 1))
        gctx = ok(d.cuGreenCtxCreate(desc, dev, d.CUgreenCtxCreate_flags.CU_GREEN_CTX_DEFAULT_STREAM))
        gst = ok(d.cuGreenCtxStreamCreate(gctx, d.CUstream_flags.CU_STREAM_NON_BLOCKING, 0))
        got_sm = ok(d.cuGreenCtxGetDevResource(gctx, d.CUdevResourceType.CU_DEV_RESOURCE_TYPE_SM))
        ctx = ok(d.cuCtxFromGreenCtx(gctx))
        ok(d.cuCtxSetCurrent(ctx))
        try:
            sp = int(gst)
            for _ in range(2):
                uz.compress(x, out=out, out_bytes=nb, stream=sp, ws=ws)
            ok(d.cuStreamSynchronize(gst))
            e0, e1 = ok(d.cuEventCreate(0)), ok(d.cuEventCreate(0))
            ok(d.cuEventRecord(e0, gst))
            for _ in range(args.steps):
                uz.compress(x, out=out, out_bytes=nb, stream=sp, ws=ws)
            ok(d.cuEventRecord(e1, gst))
            ok(d.cuEventSynchronize(e1))
            ms = ok(d.cuEventElapsedTime(e0, e1)) / args.steps
            res[f"green_ctx_{k}sm"] = {"sms": int(got_sm.sm.smCount), "compress_GBps_uncompressed":
                                       round(raw / (ms / 1e3) / GB, 2), "ms": round(ms, 4)}
        finally:
            ok(d.cuCtxSetCurrent(prim))
            d.cuGreenCtxDestroy(gctx)
    return res


if __name__ == "__main__":
    main()
