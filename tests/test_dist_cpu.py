"""Multi-process host logic on CPU (gloo, world_size 2, 127.0.0.1).

Covers the N > 1 plumbing that does not need a GPU:
  * the bootstrap all-gather callback that uzip_comm_init calls (the exact
    ctypes function the binding hands to libuzip.so), across 2 processes;
  * the CPU collective oracle run as 2 ranks exchanging inputs over gloo:
    every rank's reduce-scatter shard and allgather result equal the
    single-process oracle (the contract the GPU collectives are held to).
"""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2604_17172_b200 as uz
        import oracle
        import synth
        oracle.build()
        # 1. bootstrap callback: 72-byte "cards" (the size uzip_comm_init exchanges)
        cb = uz.torch_bootstrap(None)
        nbytes = 72
        mine = bytes((rank * 31 + i) & 0xFF for i in range(nbytes))
        src = ctypes.create_string_buffer(mine, nbytes)
        dst = ctypes.create_string_buffer(world * nbytes)
        rc = cb(ctypes.cast(src, ctypes.c_void_p), ctypes.cast(dst, ctypes.c_void_p), nbytes, None)
        assert rc == 0
        expect = b"".join(bytes((r * 31 + i) & 0xFF for i in range(nbytes)) for r in range(world))
        assert dst.raw == expect
        # 2. collective oracle across ranks
        n = 2 * 4096 + 6
        x = synth.weights(world * n, 70 + rank)
        parts = [torch.empty(world * n, dtype=torch.int32) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(x.astype(np.int32)))
        ins = [p.numpy().astype(np.uint16) for p in parts]
        assert np.array_equal(ins[rank], x)
        rs = oracle.reduce_scatter(oracle.BF16, ins, world)[rank]
        ar = oracle.allreduce(oracle.BF16, ins)
        assert np.array_equal(rs, ar[rank * n:(rank + 1) * n])
        ag = oracle.allgather(oracle.BF16, [a[:n] for a in ins])
        assert np.array_equal(ag[rank * n:(rank + 1) * n], x[:n])
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))


def test_gloo_world2_bootstrap_and_collective_oracle():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res
