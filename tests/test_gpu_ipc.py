"""CUDA-IPC (multi-process) communicator path: 2 processes on one GPU via torchrun."""
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ipc_two_processes_same_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2604_17172_b200 as uz
    uz.build()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29533", os.path.join(ROOT, "tests", "mp", "ipc_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "rank 0 ok" in r.stdout and "rank 1 ok" in r.stdout


def test_bench_dist_smoke_two_processes_same_gpu():
    """bench.py's N > 1 leg (bench_dist.py) end to end, 2 ranks time-sliced on one GPU over gloo."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json
    env = dict(os.environ, UZIP_BENCH_SMOKE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", "--master-port=29534", os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "2", "--warmup", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["compression_ratio"] < 0.75
    # the BASELINE configs[1..4] sweeps the driver's multi-GPU run reports
    su = line["suites"]
    for k in ("c2_grid", "c4_allreduce", "c5_ag_rs", "kv_p2p", "c3_weight_sync"):
        assert k in su and "skipped" not in su[k] and "error" not in su[k], (k, su.get(k))
    assert su["c2_grid"]["B4096_chunk64MiB"] > 0 and su["kv_p2p"]["per_layer"]["uzip_GBps"] > 0
    assert any(v["uzip_GBps"] for k, v in su["c5_ag_rs"].items() if k.startswith("reduce_scatter"))
    assert line["versions"]["nccl"] and "transfer_frac" in line["roofline"]


def test_protocol_under_random_delays():
    """Race shake-out: the loopback collectives re-run with UZIP_STRESS, which injects
    pseudo-random pauses of up to ~16 us before tile-flag releases and tile acquires."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, UZIP_STRESS="4242")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_comm.py"), "-k",
           "p2p_many_rounds or allgather or allreduce or broadcast or alltoall or reduce_scatter"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


_SERIAL_SCRIPT = r"""
import sys, time
sys.path.insert(0, %(root)r)
import torch
import __graft_entry__ as g
import paper_2604_17172_b200 as uz
g.smoke()  # codec round trip + one P2P round: no co-scheduled kernels needed
comms = uz.Comm.init_all(2, [0, 0], min_compress_bytes=1, staging_bytes=16 << 20)
x = torch.zeros(1 << 20, dtype=torch.bfloat16, device="cuda")
t0 = time.time()
try:
    comms[0].all_reduce(torch.empty_like(x), x)
    raise SystemExit("allreduce between co-resident ranks was not refused under serialisation")
except uz.UzipError as e:
    assert e.status == uz.ERR_COMM, e
assert time.time() - t0 < 5, "the refusal must not wait for a poll timeout"
print("serialized ok")
"""


@pytest.mark.parametrize("env", [{"CUDA_LAUNCH_BLOCKING": "1"}, {"UZIP_SERIALIZED": "1"}])
def test_serialized_execution_fails_fast(env):
    """Serialised kernels (CUDA_LAUNCH_BLOCKING, ncu): smoke() still passes and a collective between
    co-resident ranks returns UZIP_ERR_COMM at once instead of a poll timeout."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "-c", _SERIAL_SCRIPT % {"root": ROOT}], capture_output=True, text=True,
                       timeout=300, cwd=ROOT, env=dict(os.environ, **env))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "smoke ok" in r.stdout and "serialized ok" in r.stdout


def test_table_kernel_path_equals_oracle():
    """The A/B table build (UZIP_TABLE_KERNELS=1: k_hist + k_norm launched ahead of k_fused instead
    of the T items inside it) produces the same oracle streams on the codec and the collectives."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, UZIP_TABLE_KERNELS="1")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_codec.py"), os.path.join(ROOT, "tests", "test_gpu_comm.py"), "-k",
           "stream_bytes_equal_oracle or stream_params or wire_stream or allreduce_fused or tie"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]


def test_tile_trace_shows_overlap():
    """The tile trace (UZIP_TRACE=1) of a loopback split-send P2P: the receiver decodes tiles while the
    sender is still encoding later ones, and the one-pass allreduce releases allgather tiles while later
    tiles of its shard are still being reduced (overlap evidence)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import json
    env = dict(os.environ, UZIP_TRACE="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "overlap_trace.py"), "--mib", "64"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(r.stdout.strip().splitlines()[-1])
    assert res["tiles"] > 100 and res["receiver_tiles_done_before_sender_finished"] > 0.25
    assert res["allreduce_one_pass"]["ag_tiles_released_before_last_reduced_tile"] > 0.25


def test_paired_tile_receiver_forced_runs():
    """Paired-tile D items (decode-only receivers, runs of consecutive tiles) on small messages:
    UZIP_DEC_RUN=4 forces runs, so test_paired_tile_receiver_small pairs tiles (bf16 / f16 pairs, fp32
    one by one; chunk boundaries and raw blocks break pairs)."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, UZIP_DEC_RUN="4")
    cmd = [sys.executable, "-m", "pytest", "-q", "-x", "-p", "no:cacheprovider",
           os.path.join(ROOT, "tests", "test_gpu_comm.py"), "-k", "paired_tile_receiver_small or p2p_bit_exact"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
