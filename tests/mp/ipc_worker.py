"""Multi-process worker for tests/test_gpu_ipc.py (run under torchrun).

Exercises the CUDA-IPC communicator path (uzip_comm_init with a
torch.distributed bootstrap) with every rank on the SAME GPU (the only
configuration a 1-GPU box offers): the peers' regions are opened with
cudaIpcOpenMemHandle exactly as across NVLink, flags and credits cross
process boundaries.  Kernels of different processes time-slice on one GPU,
so messages are small and the poll timeout generous.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2604_17172_b200 as uz  # noqa: E402
import synth  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    comm = uz.Comm.from_group(None, 0, min_compress_bytes=1, staging_bytes=16 << 20, max_ctas=16,
                              poll_timeout_ms=60000)
    n = (1 << 20) + 4096 * 3 + 8
    # P2P 0 -> 1 (split-send), compressed
    bits = synth.weights(n, 4242)
    x = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).cuda()
    if rank == 0:
        comm.send(x, 1)
    elif rank == 1:
        y = torch.empty_like(x)
        comm.recv(y, 0)
        torch.cuda.synchronize()
        assert np.array_equal(y.view(torch.int16).cpu().numpy().view(np.uint16), bits), "P2P mismatch"
    torch.cuda.synchronize()
    dist.barrier()
    # two-shot allreduce across processes
    ins = [synth.weights(world * 262144, 100 + r) for r in range(world)]
    a = torch.from_numpy(ins[rank].view(np.int16).copy()).view(torch.bfloat16).cuda()
    out = torch.empty_like(a)
    comm.all_reduce(out, a)
    torch.cuda.synchronize()
    assert comm.async_error() == 0
    ref = oracle.allreduce(oracle.BF16, ins)
    assert np.array_equal(out.view(torch.int16).cpu().numpy().view(np.uint16), ref), "allreduce mismatch"
    dist.barrier()
    comm.destroy()
    dist.destroy_process_group()
    print(f"rank {rank} ok")


if __name__ == "__main__":
    main()
