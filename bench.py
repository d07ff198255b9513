"""bench.py -- uzip-b200 benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl uzip|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (N > 1)

Metric (BASELINE.json): effective uncompressed GB/s = raw bytes / time (GB = 1e9 B,
SURVEY 8(d)), plus the compression ratio.

N = 1 workload "c2_shard_codec_roundtrip": one step = the single-GPU part of
BASELINE configs[1] -- the 1 GiB bf16 N(0, 0.02) weight shard compressed
(uzip_compress: k_hist + k_norm + k_fused, rows a1-a5) and decompressed
(uzip_decompress: k_decode, rows a7-a8) through the C ABI.  Inputs (1 GiB) are
larger than L2 (126 MB), so no flush is needed between steps.

N > 1 workload "c2_p2p_pairs" (one process per GPU): ranks (2i, 2i+1) run the
split-send P2P of a 1 GiB bf16 shard 2i -> 2i+1 (uzip_send / uzip_recv, rows
a1-a8, a12); value = raw bytes all pairs moved / max-over-ranks time (weak).

--impl reference: the CPU oracle (oracle/, the only reference this tier has)
on a bounded sample of the same workload, timed on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GB = 1e9
BF16 = 0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="uzip", choices=["uzip", "reference"])
    ap.add_argument("--bytes", type=int, default=1 << 30, help="raw bytes per message (default 1 GiB)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-loopback", action="store_true", help="skip the loopback P2P context field (e.g. under ncu)")
    ap.add_argument("--no-dtypes", action="store_true", help="skip the per-dtype U[-1,1] context field (e.g. under ncu)")
    ap.add_argument("--no-c1", action="store_true", help="skip the C1 4 MiB latency context field (e.g. under ncu)")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: an NVML polling thread (~1 ms
    period; its first sample is taken before __enter__ returns and discarded, so every kept sample lies
    inside the with-block), falling back to `nvidia-smi -lms 100` when NVML is unavailable."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.nvml = None
        self.run = False

    def _nvml_handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
        bits = [pynvml.nvmlClocksEventReasonHwSlowdown, pynvml.nvmlClocksEventReasonHwThermalSlowdown,
                pynvml.nvmlClocksEventReasonSwThermalSlowdown, pynvml.nvmlClocksEventReasonSwPowerCap]
        return pynvml, h, bits

    def _poll(self):
        nv, h, bits = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        while self.run:
            sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
            self.rows.append([str(sm), str(mx)] + ["Active" if rs & b else "Not Active" for b in bits])
            time.sleep(0.001)

    def __enter__(self):
        try:
            self.nvml = self._nvml_handle()
            self.run = True
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            while not self.rows:
                time.sleep(0.0005)
            self.rows.clear()  # keep only samples taken inside the with-block
            return self
        except Exception:
            self.nvml, self.run = None, False
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.nvml:
            self.run = False
            self.t.join(timeout=2)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows), "source": "nvml" if self.nvml else "nvidia-smi"}


# ----------------------------------------------------------------------------- cpu baseline
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(sample_bytes: int = 1 << 30, seed: int = 1001):
    """The oracle as it stands on the same 1 GiB W workload: (1) single-threaded, pinned to one host
    core (os.sched_setaffinity), the whole 1 GiB as one stream (~10 s); (2) the same oracle functions
    fanned out over all host cores, one thread per independent 8 MiB slice (ctypes releases the GIL),
    SURVEY 8(d) "How the oracle is timed"."""
    import concurrent.futures as cf
    import numpy as np
    import oracle
    import synth
    oracle.build()
    n = sample_bytes // 2
    bits = synth.weights(n, seed)
    cores = sorted(os.sched_getaffinity(0))
    pin = cores[-1]
    try:
        os.sched_setaffinity(0, {pin})
        t0 = time.perf_counter()
        s = oracle.compress(BF16, bits)
        st, back = oracle.decompress(s, n, BF16)
        dt = time.perf_counter() - t0
    finally:
        os.sched_setaffinity(0, set(cores))
    assert st == 0 and np.array_equal(back, bits)
    slice_el = (8 << 20) // 2
    parts = [bits[i:i + slice_el] for i in range(0, n, slice_el)]

    def one(a):
        blob = oracle.compress(BF16, a)
        st2, b2 = oracle.decompress(blob, a.size, BF16)
        assert st2 == 0 and np.array_equal(b2, a)
        return len(blob)

    t0 = time.perf_counter()
    with cf.ThreadPoolExecutor(max_workers=len(cores)) as ex:
        sizes = list(ex.map(one, parts))
    dt_all = time.perf_counter() - t0
    return {"value": round(sample_bytes / dt / GB, 5), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"{sample_bytes >> 20} MiB bf16 N(0,0.02) compress+decompress, single-threaded C oracle "
                      f"pinned to core {pin}",
            "seconds": round(dt, 3), "ratio": round(len(s) / sample_bytes, 5), "cpu_model": cpu_model(),
            "all_cores": {"value": round(sample_bytes / dt_all / GB, 5), "unit": "GB/s", "cores": len(cores),
                          "kind": "oracle", "seconds": round(dt_all, 3),
                          "ratio": round(sum(sizes) / sample_bytes, 5),
                          "sample": f"{sample_bytes >> 20} MiB as {len(parts)} independent 8 MiB streams, "
                                    f"one oracle call per slice on a {len(cores)}-thread pool"}}


def reference_arm(args):
    """--impl reference: the CPU oracle on a bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numpy as np
    import oracle
    import synth
    oracle.build()
    sample = 64 << 20
    n = sample // 2
    bits = synth.weights(n, 1001)
    for _ in range(args.warmup):
        oracle.decompress(oracle.compress(BF16, bits), n, BF16)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        s = oracle.compress(BF16, bits)
        st, back = oracle.decompress(s, n, BF16)
        times.append(time.perf_counter() - t0)
        assert st == 0
    ms = 1e3 * sum(times) / len(times)
    val = sample / (ms / 1e3) / GB
    line = {"impl": "reference", "metric": "effective uncompressed GB/s", "value": round(val, 5), "unit": "GB/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic", "config": config_for(args, sample_note=f"{sample >> 20} MiB sample per step"),
            "cpu_baseline": {"value": round(val, 5), "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"{sample >> 20} MiB bf16 W compress+decompress per step"},
            "e2e": {"value": round(val, 5), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "compression_ratio": round(len(s) / sample, 5)}
    print(json.dumps(line), flush=True)


def config_for(args, sample_note=None):
    if args.gpus == 1:
        c = {"workload": "c2_shard_codec_roundtrip", "message_bytes": args.bytes, "dtype": "bf16",
             "data": "W = bf16(N(0,0.02))", "l2": "inputs 1 GiB > L2 126 MB, no flush",
             "parallelism": "single GPU"}
    else:
        c = {"workload": "c2_p2p_pairs", "message_bytes": args.bytes, "dtype": "bf16",
             "data": "W = bf16(N(0,0.02))", "l2": "inputs 1 GiB > L2 126 MB, no flush",
             "parallelism": f"{args.gpus // 2} split-send pairs"}
    if sample_note:
        c["sample"] = sample_note
    return c


# ----------------------------------------------------------------------------- uzip arm, N = 1
def run_codec(args):
    import torch
    import paper_2604_17172_b200 as uz
    uz.build()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    n = args.bytes // 2
    g = torch.Generator(device="cuda")
    g.manual_seed(1001)
    x = (torch.randn(n, device=dev, generator=g) * 0.02).to(torch.bfloat16)
    cap = uz.compress_bound(n, uz.BF16)
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    nbytes = torch.zeros(1, dtype=torch.int64, device=dev)
    y = torch.empty_like(x)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.Stream(dev)
    ws = uz.Workspace(0).get(uz.workspace_bytes(n, uz.BF16), stream)
    torch.cuda.synchronize()

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        uz.compress(x, out=out, out_bytes=nbytes, stream=stream, ws=ws)
        if ev is not None:
            ev[1].record(stream)
        uz.decompress(out, n, uz.BF16, out=y, status=st, stream=stream, ws=ws)
        if ev is not None:
            ev[2].record(stream)

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()
    assert int(st.item()) == 0 and torch.equal(x.view(torch.int16), y.view(torch.int16)), "round trip failed"
    total = int(nbytes.item())
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        start.record(stream)
        for i in range(args.steps):
            step(evs[i])
        stop.record(stream)
        torch.cuda.synchronize()
    ms = start.elapsed_time(stop) / args.steps
    enc_ms = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
    dec_ms = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
    assert int(st.item()) == 0
    raw = n * 2
    r = total / raw
    hbm, src = peaks()
    enc_bytes = raw + total           # read input, write stream (algorithmic)
    dec_bytes = total + raw           # read stream, write output
    enc_gbs = enc_bytes / (enc_ms / 1e3) / GB
    dec_gbs = dec_bytes / (dec_ms / 1e3) / GB
    dom = ("k_fused (uzip_compress; tables by its T items)", enc_gbs, enc_bytes) if enc_ms >= dec_ms else \
        ("k_decode (uzip_decompress)", dec_gbs, dec_bytes)
    traffic = ncu_traffic(["k_hist", "k_norm", "k_fused"] if enc_ms >= dec_ms else ["k_decode"], args.bytes)

    # memcpy reference on the same box (context): torch copy_ of the same bytes
    z = torch.empty_like(x)
    for _ in range(3):
        z.copy_(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        z.copy_(x)
    e1.record()
    torch.cuda.synchronize()
    copy_gbs = 2 * raw / (e0.elapsed_time(e1) / 5 / 1e3) / GB

    c1 = None if args.no_c1 else run_c1(uz)  # right after the timed region, before the heavier context legs
    e2e = None
    if not args.no_e2e:
        e2e = run_codec_e2e(uz, x, args, stream)
    loop = None if args.no_loopback else run_loopback_p2p(uz, x, args)
    per_dtype = None if args.no_dtypes else run_per_dtype(uz, args)

    line = {
        "metric": "effective uncompressed GB/s", "value": round(raw / (ms / 1e3) / GB, 3), "unit": "GB/s",
        "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic", "config": config_for(args),
        "compression_ratio": round(r, 5),
        "encode": {"ms": round(enc_ms, 4), "uncompressed_GBps": round(raw / (enc_ms / 1e3) / GB, 2),
                   "hbm_GBps": round(enc_gbs, 1), "hbm_frac": round(enc_gbs / hbm, 4)},
        "decode": {"ms": round(dec_ms, 4), "uncompressed_GBps": round(raw / (dec_ms / 1e3) / GB, 2),
                   "hbm_GBps": round(dec_gbs, 1), "hbm_frac": round(dec_gbs / hbm, 4)},
        "roofline": {"bound": "hbm", "kernel": dom[0], "achieved": round(dom[1], 1), "peak": hbm,
                     "peak_source": src, "unit": "GB/s", "frac": round(dom[1] / hbm, 4), "traffic": traffic,
                     "algorithmic_bytes_per_launch": dom[2]},
        "torch_copy_GBps": round(copy_gbs, 1),
        "loopback_p2p": loop,
        "per_dtype_uniform": per_dtype,
        "clocks": clk.summary(),
        "gpu_launches": launches_per_roundtrip(args.bytes) * args.steps,
        "c1_4mib": c1,
    }
    if e2e:
        line["e2e"] = e2e
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)


def launches_per_roundtrip(nbytes: int) -> int:
    """Our kernels per compress + decompress of a bf16 message: k_fused (its T items build the tables,
    csrc/api.cu table_kernels) + k_decode; UZIP_TABLE_KERNELS=1 adds the k_hist and k_norm launches."""
    del nbytes
    return 4 if os.environ.get("UZIP_TABLE_KERNELS", "0") != "0" else 2


def run_c1(uz, reps: int = 200):
    """BASELINE configs[0] (C1): one 4 MiB bf16 N(0,0.02) tensor compressed and decompressed -- the
    latency-bound case of P:208-210.  Mean microseconds per call over `reps` back-to-back calls
    on one stream (CUDA events), and the same for a torch copy_ of 4 MiB (the memcpy floor)."""
    import torch
    n = 2 * (1 << 20)
    g = torch.Generator(device="cuda")
    g.manual_seed(1000)
    x = (torch.randn(n, device="cuda", generator=g) * 0.02).to(torch.bfloat16)
    cap = uz.compress_bound(n, uz.BF16)
    buf = torch.empty(cap, dtype=torch.uint8, device="cuda")
    nb = torch.zeros(1, dtype=torch.int64, device="cuda")
    y = torch.empty_like(x)
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    stream = torch.cuda.Stream()
    ws = uz.Workspace(0).get(uz.workspace_bytes(n, uz.BF16), stream)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    with torch.cuda.stream(stream):
        for _ in range(10):
            uz.compress(x, out=buf, out_bytes=nb, stream=stream, ws=ws)
            uz.decompress(buf, n, uz.BF16, out=y, status=st, stream=stream, ws=ws)
        ev[0].record(stream)
        for _ in range(reps):
            uz.compress(x, out=buf, out_bytes=nb, stream=stream, ws=ws)
        ev[1].record(stream)
        for _ in range(reps):
            uz.decompress(buf, n, uz.BF16, out=y, status=st, stream=stream, ws=ws)
        ev[2].record(stream)
        z = torch.empty_like(x)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            z.copy_(x)
        e1.record(stream)
    torch.cuda.synchronize()
    ok = int(st.item()) == 0 and torch.equal(x.view(torch.int16), y.view(torch.int16))
    cu = ev[0].elapsed_time(ev[1]) * 1e3 / reps
    du = ev[1].elapsed_time(ev[2]) * 1e3 / reps
    ok = ok and int(st.item()) == 0 and torch.equal(x.view(torch.int16), y.view(torch.int16))
    return {"bytes": 2 * n, "compress_us": round(cu, 2), "decompress_us": round(du, 2),
            "roundtrip_GBps": round(2 * n / ((cu + du) * 1e-6) / GB, 1), "ratio": round(int(nb.item()) / (2 * n), 5),
            "copy_us": round(e0.elapsed_time(e1) * 1e3 / reps, 2), "bit_exact": bool(ok),
            "launches_per_roundtrip": launches_per_roundtrip(2 * n),
            "note": "back-to-back calls on one stream, CUDA events; the Python + C host path issues a call in "
                    "~17 us (scripts/c1_host.py), below the device time, so the numbers are device-bound"}


def run_per_dtype(uz, args):
    """Context (the paper's per-dtype table): ratio and round-trip GB/s of 256 MiB of
    U[-1,1] (the paper's synthetic input) per dtype; paper ratios f16 0.83, f32 0.82,
    bf16 0.64, e4m3 0.77, e5m2 0.70."""
    import torch
    out = {}
    nbytes = 256 << 20
    g = torch.Generator(device="cuda")
    for name, tdt, paper in (("bf16", torch.bfloat16, 0.64), ("f16", torch.float16, 0.83),
                             ("f32", torch.float32, 0.82), ("e4m3", torch.float8_e4m3fn, 0.77),
                             ("e5m2", torch.float8_e5m2, 0.70)):
        g.manual_seed(7)
        n = nbytes // torch.tensor([], dtype=tdt).element_size()
        x = (torch.rand(n, device="cuda", generator=g) * 2 - 1).to(tdt)
        dt = uz.uz_dtype(tdt)
        cap = uz.compress_bound(n, dt)
        buf = torch.empty(cap, dtype=torch.uint8, device="cuda")
        nb = torch.zeros(1, dtype=torch.int64, device="cuda")
        y = torch.empty_like(x)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        ws = uz.Workspace(0).get(uz.workspace_bytes(n, dt))
        for _ in range(2):
            uz.compress(x, out=buf, out_bytes=nb, ws=ws)
            uz.decompress(buf, n, dt, out=y, status=st, ws=ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            uz.compress(x, out=buf, out_bytes=nb, ws=ws)
            uz.decompress(buf, n, dt, out=y, status=st, ws=ws)
        e1.record()
        torch.cuda.synchronize()
        ok = int(st.item()) == 0 and torch.equal(x.view(torch.uint8), y.view(torch.uint8))
        out[name] = {"ratio": round(int(nb.item()) / nbytes, 4), "paper_ratio": paper,
                     "roundtrip_GBps": round(nbytes / (e0.elapsed_time(e1) / 5 / 1e3) / GB, 1), "bit_exact": ok}
    return out


def run_loopback_p2p(uz, x, args):
    """Context (not the headline): the full split-send path -- uzip_send on rank 0 and uzip_recv on
    rank 1 -- with both ranks on this one GPU (loopback communicators), each persistent kernel capped
    at half the SM slots.  Sender and receiver share the SMs and HBM, so this is a lower bound for
    the NVLink case; the bytes still go through staging, tile flags and credits."""
    import torch
    comms = uz.Comm.init_all(2, [0, 0], max_ctas=2 * 148, staging_bytes=1 << 30)
    s0, s1 = torch.cuda.Stream(), torch.cuda.Stream()
    y = torch.empty_like(x)

    def step():
        s1.wait_stream(s0)
        comms[0].send(x, 1, s0)
        comms[1].recv(y, 0, s1)
        s0.wait_stream(s1)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s0)
    for _ in range(args.steps):
        step()
    e1.record(s0)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    errs = [c.async_error() for c in comms]
    ok = torch.equal(x.view(torch.int16), y.view(torch.int16)) and errs == [0, 0]
    st = comms[0].stats()
    for c in comms:
        c.destroy()
    return {"value": round(x.numel() * 2 / (ms / 1e3) / GB, 2), "unit": "GB/s", "ms": round(ms, 4),
            "bit_exact": bool(ok), "async_errors": errs,
            "wire_ratio": round(st["wire_bytes"] / max(1, st["raw_bytes"]), 5),
            "note": "sender+receiver kernels share one GPU (loopback), 1 GiB bf16 W"}


def ncu_traffic(kernels, nbytes):
    """DRAM bytes (read + write) per launch of the named kernels from the latest committed ncu
    `--set full` capture (profiles/*_traffic.json, written by scripts/ncu_summary.py for the same
    1 GiB bench command); None when absent or taken at another size."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_traffic.json")))
    if not files or nbytes != 1 << 30:
        return None
    d = json.load(open(files[-1]))
    vals = [v for k, v in d.items() for name in kernels if name in k]
    return int(sum(vals)) if vals else None


def run_codec_e2e(uz, x, args, stream):
    """Same metric through the public API with host buffers: every step copies its input H2D from
    pinned host memory, compresses, decompresses and copies the decompressed result + status D2H.
    Steps are pipelined over two buffer sets and three streams (H2D, compute, D2H), so step i+1's
    H2D and step i-1's D2H (the two PCIe directions) overlap step i's compute; the timed region spans
    all steps, from the first H2D to the last D2H (host clock, synchronized on both sides)."""
    import torch
    n = x.numel()
    dev = x.device
    nbuf = 2
    host_in = [torch.empty(n, dtype=torch.bfloat16, pin_memory=True) for _ in range(nbuf)]
    host_in[0].copy_(x.cpu())
    host_in[1].copy_(host_in[0].view(torch.int16).flip(0).view(torch.bfloat16))  # a second message
    back = [torch.empty(n, dtype=torch.bfloat16, pin_memory=True) for _ in range(nbuf)]
    res_h = [torch.empty(2, dtype=torch.int64, pin_memory=True) for _ in range(nbuf)]
    xd = [torch.empty_like(x) for _ in range(nbuf)]
    y = [torch.empty_like(x) for _ in range(nbuf)]
    res_d = [torch.empty(2, dtype=torch.int64, device=dev) for _ in range(nbuf)]
    cap = uz.compress_bound(n, uz.BF16)
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    nbytes = torch.zeros(1, dtype=torch.int64, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = uz.Workspace(0).get(uz.workspace_bytes(n, uz.BF16), stream)
    s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev = lambda: torch.cuda.Event()  # noqa: E731
    h2d_done = [ev() for _ in range(nbuf)]
    comp_done = [ev() for _ in range(nbuf)]   # compute finished reading xd[k] and writing y[k]
    d2h_done = [ev() for _ in range(nbuf)]    # y[k] / res_d[k] copied out
    for k in range(nbuf):
        comp_done[k].record(stream)
        d2h_done[k].record(s_d2h)

    def issue(i):
        k = i % nbuf
        s_h2d.wait_event(comp_done[k])  # xd[k] free (step i-2's compress has read it)
        with torch.cuda.stream(s_h2d):
            xd[k].copy_(host_in[k], non_blocking=True)
            h2d_done[k].record(s_h2d)
        stream.wait_event(h2d_done[k])
        stream.wait_event(d2h_done[k])  # y[k] free (step i-2's result is on the host)
        with torch.cuda.stream(stream):
            uz.compress(xd[k], out=out, out_bytes=nbytes, stream=stream, ws=ws)
            uz.decompress(out, n, uz.BF16, out=y[k], status=st, stream=stream, ws=ws)
            res_d[k][0:1].copy_(nbytes)
            res_d[k][1:2].copy_(st)
            comp_done[k].record(stream)
        s_d2h.wait_event(comp_done[k])
        with torch.cuda.stream(s_d2h):
            res_h[k].copy_(res_d[k], non_blocking=True)
            back[k].copy_(y[k], non_blocking=True)  # the round trip's result returns to the host
            d2h_done[k].record(s_d2h)

    for i in range(2 * nbuf):  # warm-up
        issue(i)
    torch.cuda.synchronize(dev)
    steps = max(4, args.steps)
    t0 = time.perf_counter()
    for i in range(steps):
        issue(i)
    torch.cuda.synchronize(dev)
    dt = (time.perf_counter() - t0) / steps
    for k in range(nbuf):
        assert int(res_h[k][1]) == 0 and torch.equal(back[k].view(torch.int16), host_in[k].view(torch.int16))
    return {"value": round(2 * n / dt / GB, 3), "unit": "GB/s", "h2d_bytes_per_step": 2 * n,
            "d2h_bytes_per_step": 2 * n + 16, "ms_per_step": round(dt * 1e3, 3),
            "note": "per step: pinned H2D of the input, compress, decompress, D2H of the decompressed output + "
                    "status; steps pipelined over 2 buffer sets and H2D / compute / D2H streams (the two PCIe "
                    "directions overlap), all steps inside the timed region; PCIe-bound"}


def main():
    args = parse()
    if args.impl == "reference":
        reference_arm(args)
        return
    if args.gpus == 1 and int(os.environ.get("WORLD_SIZE", "1")) == 1:
        run_codec(args)
    else:
        import bench_dist
        bench_dist.run(args)


if __name__ == "__main__":
    main()
