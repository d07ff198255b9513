"""bench_dist.py -- the N > 1 leg of bench.py (one process per GPU under torchrun).

Workload "c2_p2p_pairs": ranks (2i, 2i+1) run the split-send P2P of a 1 GiB
bf16 N(0, 0.02) shard 2i -> 2i+1 through uzip_send / uzip_recv (BASELINE
configs[1]); value = raw bytes all pairs moved per second, timed on the device
(CUDA events on each rank's stream, barrier + synchronize on both sides, max
over ranks).  Alongside: the same transfer through NCCL send/recv on the same
buffers, and the two-shot compressed allreduce of a 256 MiB bf16 activation
tensor (configs[3]) against NCCL all_reduce.
"""
from __future__ import annotations

import json
import os
import statistics
import time

import torch
import torch.distributed as dist

GB = 1e9


SMOKE = os.environ.get("UZIP_BENCH_SMOKE") == "1"  # 2 ranks on one GPU over gloo: code-path check only


def _max_over_ranks(v: float) -> float:
    t = torch.tensor([v], device="cpu" if SMOKE else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _timed(fn, stream, steps, warmup, group=None):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier(group)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = _max_over_ranks(e0.elapsed_time(e1))
    dist.barrier(group)
    return ms / steps


def run(args):
    import bench
    import paper_2604_17172_b200 as uz

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = 0 if SMOKE else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if SMOKE:
        dist.init_process_group("gloo")
        args.bytes = min(args.bytes, 8 << 20)
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    uz.build() if rank == 0 else None
    dist.barrier()
    comm = uz.Comm.from_group(None, local, **(dict(staging_bytes=32 << 20, max_ctas=16, poll_timeout_ms=60000)
                                              if SMOKE else {}))
    stream = torch.cuda.Stream()
    n = args.bytes // 2
    g = torch.Generator(device="cuda")
    g.manual_seed(1001 + rank)
    x = (torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    y = torch.empty_like(x)
    pairs = world // 2
    raw = pairs * 2 * n
    role = "send" if rank % 2 == 0 and rank + 1 < world else ("recv" if rank % 2 == 1 else "idle")
    peer = rank + 1 if role == "send" else rank - 1

    def uz_step():
        with torch.cuda.stream(stream):
            if role == "send":
                comm.send(x, peer, stream)
            elif role == "recv":
                comm.recv(y, peer, stream)

    def nccl_step():
        with torch.cuda.stream(stream):
            if role == "send":
                dist.send(x, peer)
            elif role == "recv":
                dist.recv(y, peer)

    with bench.ClockSampler(local) as clk:
        ms = _timed(uz_step, stream, args.steps, args.warmup)
    assert comm.async_error() == 0
    st = comm.stats() if role == "send" else None
    # correctness spot check: receiver sees the sender's bytes
    if role == "send":
        dist.send(x.cpu() if SMOKE else x, peer)
    elif role == "recv":
        ref = torch.empty(x.shape, dtype=x.dtype, device="cpu" if SMOKE else x.device)
        dist.recv(ref, peer)
        assert torch.equal(ref.view(torch.int16).cpu(), y.view(torch.int16).cpu()), "P2P mismatch"
    ms_nccl = float("nan") if SMOKE else _timed(nccl_step, stream, args.steps, args.warmup)

    # ablation (fig:compare_with_native_pipeline): encode-send = compress the whole
    # message, ship the stream with NCCL, decompress -- no overlap, no fused transfer
    ablation = {}
    if not SMOKE:
        cap = uz.compress_bound(n, uz.BF16)
        sbuf = torch.empty(cap, dtype=torch.uint8, device="cuda")
        nb = torch.zeros(1, dtype=torch.int64, device="cuda")
        stat = torch.zeros(1, dtype=torch.int32, device="cuda")
        ws = uz.Workspace(local).get(uz.workspace_bytes(n, uz.BF16), stream)
        with torch.cuda.stream(stream):
            if role == "send":
                uz.compress(x, out=sbuf, out_bytes=nb, stream=stream, ws=ws)
        torch.cuda.synchronize()
        szt = nb.clone()
        if role == "send":
            dist.send(szt, peer)  # the stream size is deterministic for this input: exchanged once
        elif role == "recv":
            dist.recv(szt, peer)
        wire = int(szt.item())

        def encode_send():
            with torch.cuda.stream(stream):
                if role == "send":
                    uz.compress(x, out=sbuf, out_bytes=nb, stream=stream, ws=ws)
                    dist.send(sbuf[:wire], peer)
                elif role == "recv":
                    dist.recv(sbuf[:wire], peer)
                    uz.decompress(sbuf, n, uz.BF16, out=y, status=stat, stream=stream, ws=ws, in_bytes=wire)

        ms_es = _timed(encode_send, stream, args.steps, args.warmup)
        ablation = {"encode_send_GBps": round(raw / (ms_es / 1e3) / GB, 3), "ms": round(ms_es, 4),
                    "note": "uzip_compress + NCCL send of the stream + uzip_decompress, serial"}

        # chunked pipeline (one stream and one launch per 8 MiB chunk) and SM-limited runs
        # (fig:resource_usage; a CTA cap per side stands in for Green Contexts): same calls, other configs
        def p2p_with(**cfg):
            cm = uz.Comm.from_group(None, local, **cfg)

            def step():
                with torch.cuda.stream(stream):
                    if role == "send":
                        cm.send(x, peer, stream)
                    elif role == "recv":
                        cm.recv(y, peer, stream)
            t = _timed(step, stream, args.steps, args.warmup)
            assert cm.async_error() == 0
            cm.destroy()
            return round(raw / (t / 1e3) / GB, 3)

        ablation["chunked_8MiB_GBps"] = p2p_with(pipe_chunk_bytes=8 << 20)
        ablation["block_sweep_GBps"] = {str(bs): p2p_with(block_symbols=bs) for bs in (1024, 2048)}  # 4096: value
        ablation["sm_limited_GBps"] = {str(m): p2p_with(max_ctas=m) for m in (16, 37, 74, 148)}

    # e2e through the public API with host buffers: the sender copies its input from pinned host memory
    # and sends; the receiver receives and reads 16 bytes of the result back; wall clock, max over ranks
    host = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
    if role == "send":
        host.copy_(x.cpu())
    xd = torch.empty_like(x)
    res_h = torch.empty(8, dtype=torch.int16, pin_memory=True)

    def e2e_step():
        with torch.cuda.stream(stream):
            if role == "send":
                xd.copy_(host, non_blocking=True)
                comm.send(xd, peer, stream)
            elif role == "recv":
                comm.recv(y, peer, stream)
                res_h.copy_(y[:8].view(torch.int16), non_blocking=True)
        stream.synchronize()

    for _ in range(args.warmup):
        e2e_step()
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        e2e_step()
    e2e_s = _max_over_ranks(time.perf_counter() - t0) / args.steps
    dist.barrier()

    # collectives on the same box, uzip vs NCCL (algbw = user bytes / time, nccl-tests convention)
    MB = 1 << 20
    T = ((8 if SMOKE else 256) * MB) // (2 * 4096)
    ga = torch.Generator(device="cuda")
    ga.manual_seed(3000 + rank)
    scale = torch.exp(torch.randn(4096, device="cuda", generator=ga) * 0.5)
    a = (torch.randn(T, 4096, device="cuda", generator=ga) * scale).to(torch.bfloat16)  # activations (C4)
    ar_out = torch.empty_like(a)
    nc_buf = a.clone()
    coll = {}

    def measure(name, uz_fn, nccl_fn, user_bytes):
        ms_u = _timed(uz_fn, stream, args.steps, args.warmup)
        stt = comm.stats()
        ms_n = float("nan") if SMOKE else _timed(nccl_fn, stream, args.steps, args.warmup)
        coll[name] = {"uzip_algbw_GBps": round(user_bytes / (ms_u / 1e3) / GB, 2),
                      "nccl_algbw_GBps": round(user_bytes / (ms_n / 1e3) / GB, 2), "ms": round(ms_u, 4),
                      "ms_nccl": round(ms_n, 4),
                      "wire_ratio": round(stt["wire_bytes"] / max(1, stt["raw_bytes"]), 5)}

    def in_stream(f):
        def g():
            with torch.cuda.stream(stream):
                f()
        return g

    measure("allreduce_256MiB_act", in_stream(lambda: comm.all_reduce(ar_out, a, stream)),
            in_stream(lambda: dist.all_reduce(nc_buf)), 2 * a.numel())
    shard = a.view(-1)[: a.numel() // world]
    ag_out = torch.empty(world * shard.numel(), dtype=a.dtype, device="cuda")
    measure("allgather_256MiB_out", in_stream(lambda: comm.all_gather(ag_out, shard, stream)),
            in_stream(lambda: dist.all_gather_into_tensor(ag_out, shard)), 2 * ag_out.numel())
    rs_out = torch.empty(a.numel() // world, dtype=a.dtype, device="cuda")
    measure("reduce_scatter_256MiB_in", in_stream(lambda: comm.reduce_scatter(rs_out, a.view(-1), stream)),
            in_stream(lambda: dist.reduce_scatter_tensor(rs_out, a.view(-1))), 2 * a.numel())
    wb = x if rank == 0 else y  # weight-sync broadcast of the 1 GiB W shard from rank 0 (C3 analog)
    measure("broadcast_1GiB_w", in_stream(lambda: comm.broadcast(wb, 0, stream)),
            in_stream(lambda: dist.broadcast(wb, 0)), 2 * n)
    assert comm.async_error() == 0

    # ---- BASELINE configs[1..4] sweeps, each bounded in time; results keyed by config
    suites = run_suites(args, uz, comm, stream, rank, world, local, x, y, role, peer, n)

    sts = [None] * world
    dist.all_gather_object(sts, st)
    if rank == 0:
        ratio = next((s["wire_bytes"] / s["raw_bytes"] for s in sts if s), None)
        wire_gbs = (ratio or 1.0) * 2 * n / (ms / 1e3) / GB
        hbm, _ = bench.peaks()
        r = ratio or 1.0
        S = 2 * n
        # transfer roofline (north_star): the slower of codec-at-HBM-peak (receiver: r*S written by the
        # sender + r*S read + S written; sender: S read) and the compressed bytes over one NVLink direction
        t_codec = max(S, (2 * r + 1) * S) / (hbm * GB)
        t_wire = r * S / (770.0 * GB)
        t_bound = max(t_codec, t_wire)
        line = {
            "metric": "effective uncompressed GB/s", "value": round(raw / (ms / 1e3) / GB, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": bench.config_for(args), "compression_ratio": round(ratio, 5) if ratio else None,
            "nccl_send_recv": {"value": round(raw / (ms_nccl / 1e3) / GB, 3), "unit": "GB/s",
                               "ms_per_step": round(ms_nccl, 4)},
            "collectives": coll,
            "ablation": ablation,
            "roofline": {"bound": "nvlink", "kernel": "k_fused (sender E items + receiver D items, split-send)",
                         "achieved": round(wire_gbs, 1), "peak": 770.0, "unit": "GB/s",
                         "peak_source": "B200_PROFILING.md measured peer copy per direction",
                         "frac": round(wire_gbs / 770.0, 4), "traffic": None,
                         "transfer_bound_ms": round(t_bound * 1e3, 4),
                         "transfer_frac": round(t_bound / (ms / 1e3 / max(1, pairs)) if pairs else 0.0, 4),
                         "note": "transfer_frac = max(codec at HBM peak, r*S / 770 GB/s) / time per pair"},
            "e2e": {"value": round(raw / e2e_s / GB, 3), "unit": "GB/s", "h2d_bytes_per_step": pairs * 2 * n,
                    "d2h_bytes_per_step": pairs * 16, "ms_per_step": round(e2e_s * 1e3, 3)},
            "clocks": clk.summary(),
            "gpu_launches": args.steps * 2 * 2 * max(1, (2 * n) // (256 << 20)),
            "versions": versions(),
            "suites": suites,
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()


def versions():
    import subprocess
    v = {"torch": torch.__version__, "cuda": torch.version.cuda}
    try:
        nv = torch.cuda.nccl.version()
        v["nccl"] = ".".join(map(str, nv)) if isinstance(nv, tuple) else str(nv)
    except Exception as e:  # pragma: no cover
        v["nccl"] = repr(e)[:80]
    try:
        v["driver"] = subprocess.run(["nvidia-smi", "--query-gpu=driver_version,name", "--format=csv,noheader"],
                                     capture_output=True, text=True, timeout=20).stdout.splitlines()[0].strip()
    except Exception as e:  # pragma: no cover
        v["driver"] = repr(e)[:80]
    v["NCCL_ALGO"] = os.environ.get("NCCL_ALGO", "default")
    return v


def nvlink_bytes(index):
    """(tx, rx) NVLink data bytes of GPU `index` so far, summed over its links (NVML throughput
    counters, KiB), or None where NVML or the counters are unavailable (no NVLink, one-GPU boxes)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        tx = rx = 0
        seen = False
        for link in range(18):
            try:
                if pynvml.nvmlDeviceGetNvLinkState(h, link) != pynvml.NVML_FEATURE_ENABLED:
                    continue
            except pynvml.NVMLError:
                continue
            vals = pynvml.nvmlDeviceGetFieldValues(h, [(pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, link),
                                                       (pynvml.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, link)])
            if vals[0].nvmlReturn or vals[1].nvmlReturn:
                continue
            tx += vals[0].value.ullVal * 1024
            rx += vals[1].value.ullVal * 1024
            seen = True
        return (tx, rx) if seen else None
    except Exception:
        return None


def _fill_w(buf, seed):
    """W = bf16(N(0, 0.02)) in 64 Mi-element slices (no fp32 temporary of the whole buffer)."""
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    flat = buf.view(-1)
    step = 64 << 20
    for o in range(0, flat.numel(), step):
        k = min(step, flat.numel() - o)
        flat[o:o + k].copy_(torch.randn(k, device="cuda", generator=g) * 0.02)
    return buf


def run_suites(args, uz, comm, stream, rank, world, local, x, y, role, peer, n):
    """BASELINE configs[1]-[4] as sweeps: C2 pipe-chunk x block-size grid, C3 Qwen2.5-7B
    weight sync (per tensor and 256 MiB buckets) vs NCCL broadcast, C4 activation allreduce
    256 KiB-256 MiB vs NCCL, C5 allgather / reduce-scatter 1 MiB-4 GiB vs NCCL, KV-cache P2P.
    Every entry: uzip and NCCL algbw (GB/s, nccl-tests convention) and the wire ratio.  Each suite
    is skipped once the budget (UZIP_BENCH_BUDGET_S, default 300 s) is spent; UZIP_BENCH_SUITES
    selects a comma-separated subset ("none" skips all)."""
    budget = float(os.environ.get("UZIP_BENCH_BUDGET_S", "300"))
    want = os.environ.get("UZIP_BENCH_SUITES", "c2_grid,c4_allreduce,c5_ag_rs,kv_p2p,c3_weight_sync")
    t0 = time.time()
    out = {}
    steps = max(1, min(args.steps, 2 if SMOKE else 5))
    warm = 1
    MB = 1 << 20

    def timed(fn):
        return _timed(fn, stream, steps, warm)

    def gbs(nbytes, ms_):
        return round(nbytes / (ms_ / 1e3) / GB, 2) if ms_ == ms_ and ms_ > 0 else None

    def in_stream(f):
        def g():
            with torch.cuda.stream(stream):
                f()
        return g

    def pair(uz_fn, nccl_fn, user_bytes, cm=None):
        cm = cm or comm
        mu = timed(in_stream(uz_fn))
        stt = cm.stats()
        mn = float("nan") if SMOKE or nccl_fn is None else timed(in_stream(nccl_fn))
        return {"uzip_GBps": gbs(user_bytes, mu), "nccl_GBps": gbs(user_bytes, mn), "ms": round(mu, 4),
                "ms_nccl": round(mn, 4) if mn == mn else None,
                "wire_ratio": round(stt["wire_bytes"] / max(1, stt["raw_bytes"]), 5)}

    def suite(name, fn):
        if name not in want.split(","):
            return
        if time.time() - t0 > budget:
            out[name] = {"skipped": f"time budget {budget:.0f} s spent"}
            return
        ts = time.time()
        nv0 = nvlink_bytes(local)
        out[name] = fn()
        torch.cuda.synchronize()
        dist.barrier()
        out[name]["seconds"] = round(time.time() - ts, 1)
        nv1 = nvlink_bytes(local)
        # this rank's NVLink data bytes over the whole suite (uzip and NCCL legs): counter evidence that
        # the traffic went over NVLink, not a per-leg number
        out[name]["nvlink_GB_rank"] = (None if nv0 is None or nv1 is None else
                                       {"tx": round((nv1[0] - nv0[0]) / 1e9, 3), "rx": round((nv1[1] - nv0[1]) / 1e9, 3)})

    pairs = world // 2

    def c2_grid():
        """split-send P2P of the 1 GiB shard, pairs (2i -> 2i+1): pipe chunk x codec block size."""
        res = {}
        chunks = (4, 64) if SMOKE else (4, 16, 64, 256, 1024)
        for B in ((1024, 4096, 16384) if SMOKE else (1024, 2048, 4096, 8192, 16384)):
            for pc in chunks:
                stg = max(512 * MB, 2 * pc * MB)
                cm = uz.Comm.from_group(None, local, block_symbols=B, pipe_chunk_bytes=pc * MB,
                                        staging_bytes=min(stg, 32 * MB) if SMOKE else stg,
                                        **(dict(max_ctas=16, poll_timeout_ms=60000) if SMOKE else {}))

                def step():
                    if role == "send":
                        cm.send(x, peer, stream)
                    elif role == "recv":
                        cm.recv(y, peer, stream)
                ms_ = timed(in_stream(step))
                assert cm.async_error() == 0
                res[f"B{B}_chunk{pc}MiB"] = gbs(pairs * 2 * n, ms_)
                cm.destroy()
        res["note"] = "GB/s of all pairs; B = 8192 / 16384 blocks exceed the receivers' smem staging (decoded in place)"
        return res

    def c4_allreduce():
        """Llama-3-8B TP activation allreduce, T = 32 * 2^k tokens x 4096 (256 KiB - 256 MiB)."""
        res = {}
        ks = range(0, 5) if SMOKE else range(0, 11)
        ga = torch.Generator(device="cuda")
        ga.manual_seed(3000 + rank)
        scale = torch.exp(torch.randn(4096, device="cuda", generator=ga) * 0.5)
        # NCCL with its ring algorithm forced as a second baseline (SURVEY 7 hard part 5): NCCL reads
        # NCCL_ALGO when a communicator is created, so a fresh group is built with the variable set
        ring_pg, ring_err = None, None
        if not SMOKE and os.environ.get("UZIP_BENCH_NCCL_RING", "1") != "0":
            old = os.environ.get("NCCL_ALGO")
            try:
                os.environ["NCCL_ALGO"] = "Ring"
                ring_pg = dist.new_group(backend="nccl")
                warm = torch.ones(1024, device="cuda")
                dist.all_reduce(warm, group=ring_pg)  # the communicator is created here
                torch.cuda.synchronize()
            except Exception as e:  # report, keep the suite
                ring_pg, ring_err = None, repr(e)[:200]
            finally:
                if old is None:
                    os.environ.pop("NCCL_ALGO", None)
                else:
                    os.environ["NCCL_ALGO"] = old
        for k in ks:
            T = 32 << k
            a = (torch.randn(T, 4096, device="cuda", generator=ga) * scale).to(torch.bfloat16)
            o = torch.empty_like(a)
            nb = a.clone()
            key = f"{2 * a.numel() >> 10}KiB"
            res[key] = pair(lambda: comm.all_reduce(o, a, stream), lambda: dist.all_reduce(nb), 2 * a.numel())
            if ring_pg is not None:
                try:
                    mr = timed(in_stream(lambda: dist.all_reduce(nb, group=ring_pg)))
                    res[key]["nccl_ring_GBps"] = gbs(2 * a.numel(), mr)
                except Exception as e:
                    res[key]["nccl_ring_error"] = repr(e)[:200]
        if ring_err:
            res["nccl_ring_error"] = ring_err
        return res

    def c5_ag_rs():
        """allgather (S = total output) and reduce-scatter (S = total input per rank), S = 1 MiB - 4 GiB."""
        res = {}
        top = 26 if SMOKE else 32
        big = torch.empty((1 << top) // 2, dtype=torch.bfloat16, device="cuda")
        _fill_w(big, 5000 + rank)
        for lg in range(20, top + 1):
            S = 1 << lg
            el = S // 2
            if el % (world * 8):
                continue
            shard = big[: el // world]
            agout = torch.empty(el, dtype=torch.bfloat16, device="cuda")
            res[f"allgather_{S >> 20}MiB"] = pair(lambda: comm.all_gather(agout, shard, stream),
                                                 lambda: dist.all_gather_into_tensor(agout, shard), S)
            del agout
            rsin = big[:el]
            rsout = torch.empty(el // world, dtype=torch.bfloat16, device="cuda")
            res[f"reduce_scatter_{S >> 20}MiB"] = pair(lambda: comm.reduce_scatter(rsout, rsin, stream),
                                                      lambda: dist.reduce_scatter_tensor(rsout, rsin), S)
            del rsout
        del big
        torch.cuda.empty_cache()
        return res

    def kv_p2p():
        """Llama-3-8B KV cache, 7680 tokens = 480 blocks x 32 layers x 64 KiB = 960 MiB bf16, pairs
        2i -> 2i+1: one message and 32 per-layer messages of 30 MiB."""
        layers, nb = (4, 60) if SMOKE else (32, 480)
        gk = torch.Generator(device="cuda")
        gk.manual_seed(8000 + rank)
        kscale = torch.exp(torch.randn(layers, 1, 1, 8, 128, device="cuda", generator=gk) * 0.5)
        k = torch.randn(layers, nb, 16, 8, 128, device="cuda", generator=gk) * kscale
        v = torch.randn(layers, nb, 16, 8, 128, device="cuda", generator=gk)
        kv = torch.stack([k, v], dim=2).to(torch.bfloat16).contiguous().view(layers, -1)
        del k, v
        rx = torch.empty_like(kv)
        tot = pairs * 2 * kv.numel()

        def one(u):
            if role == "send":
                (comm.send(kv.view(-1), peer, stream) if u else dist.send(kv.view(-1), peer))
            elif role == "recv":
                (comm.recv(rx.view(-1), peer, stream) if u else dist.recv(rx.view(-1), peer))

        def per_layer(u):
            for i in range(layers):
                if role == "send":
                    (comm.send(kv[i], peer, stream) if u else dist.send(kv[i], peer))
                elif role == "recv":
                    (comm.recv(rx[i], peer, stream) if u else dist.recv(rx[i], peer))
        return {"one_message": pair(lambda: one(True), lambda: one(False), tot),
                "per_layer": pair(lambda: per_layer(True), lambda: per_layer(False), tot),
                "bytes_per_pair": 2 * kv.numel()}

    def c3_weight_sync():
        """Qwen2.5-7B-shaped bf16 weights (339 tensors, 15.23 GB) broadcast from rank 0 to all others:
        per tensor and in 256 MiB buckets (uzip compressed scatter + relay vs NCCL broadcast)."""
        h, kvd, ff, vocab = 3584, 512, 18944, 152064
        layer = [(h, h), (h,), (kvd, h), (kvd,), (kvd, h), (kvd,), (h, h), (ff, h), (ff, h), (h, ff), (h,), (h,)]
        shapes = [(vocab, h)] + layer * 28 + [(h,), (vocab, h)]
        sizes = [int(torch.tensor(s).prod()) for s in shapes]
        if SMOKE:
            sizes = [max(8, s // 4096 // 8 * 8) for s in sizes[:20]]  # views stay 16-byte aligned
        total = sum(sizes)
        flat = torch.empty(total, dtype=torch.bfloat16, device="cuda")
        if rank == 0:
            _fill_w(flat, 7000)
        views, o = [], 0
        for s in sizes:
            views.append(flat[o:o + s])
            o += s
        bucket = (256 * MB) // 2
        buckets = [flat[i:i + bucket] for i in range(0, total, bucket)]
        res = {"tensors": len(sizes), "bytes": 2 * total}
        res["per_tensor"] = pair(lambda: [comm.broadcast(t, 0, stream) for t in views],
                                 lambda: [dist.broadcast(t, 0) for t in views], 2 * total)
        res["bucket_256MiB"] = pair(lambda: [comm.broadcast(t, 0, stream) for t in buckets],
                                    lambda: [dist.broadcast(t, 0) for t in buckets], 2 * total)
        del flat, views, buckets
        torch.cuda.empty_cache()
        return res

    # most informative first (the collectives vs NCCL), the 15-communicator C2 grid last
    suite("c4_allreduce", c4_allreduce)
    suite("c5_ag_rs", c5_ag_rs)
    suite("kv_p2p", kv_p2p)
    suite("c3_weight_sync", c3_weight_sync)
    suite("c2_grid", c2_grid)
    out["budget_s"] = budget
    return out
