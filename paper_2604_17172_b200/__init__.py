"""uzip-b200: Python binding of libuzip.so (include/uzip.h), argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; this module
converts torch tensors to device pointers and CUDA streams and forwards to the
C ABI.  There is no CPU fallback: if libuzip.so is missing or no CUDA device is
visible, the data calls raise.

Method: arxiv 2604.17172 ("Uzip"), §2.1.2 codec, §3.2
split-send, §3.3-3.4 fused collectives; stream format
and readings in DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import _build

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("UZIP_LIB_PATH") or os.path.join(_HERE, "libuzip.so")  # override: tuning variants

BF16, F16, F32, E4M3, E5M2 = 0, 1, 2, 3, 4
SUM, MIN, MAX = 0, 1, 2
STATUS = {0: "OK", 1: "INVALID_ARG", 2: "UNSUPPORTED_DTYPE", 3: "CAPACITY", 4: "CORRUPT_STREAM",
          5: "SIZE_MISMATCH", 6: "CUDA", 7: "COMM", 8: "TIMEOUT", 9: "NOT_IMPLEMENTED"}
OK, ERR_INVALID_ARG, ERR_UNSUPPORTED_DTYPE, ERR_CAPACITY, ERR_CORRUPT_STREAM, ERR_SIZE_MISMATCH, \
    ERR_CUDA, ERR_COMM, ERR_TIMEOUT, ERR_NOT_IMPLEMENTED = range(10)

_TORCH_TO_UZ = {torch.bfloat16: BF16, torch.float16: F16, torch.float32: F32, torch.float8_e4m3fn: E4M3,
                torch.float8_e5m2: E5M2}
_UZ_TO_TORCH = {v: k for k, v in _TORCH_TO_UZ.items()}
ELEM_BYTES = {BF16: 2, F16: 2, F32: 4, E4M3: 1, E5M2: 1}

EXPORTED = [
    "uzip_compress_bound", "uzip_workspace_bytes", "uzip_workspace_init", "uzip_compress", "uzip_decompress",
    "uzip_comm_init", "uzip_comm_init_all", "uzip_comm_destroy", "uzip_send", "uzip_recv", "uzip_allgather",
    "uzip_reduce_scatter", "uzip_allreduce", "uzip_comm_get_async_error", "uzip_get_stats",
    "uzip_status_string", "uzip_version", "uzip_comm_read_staging", "uzip_broadcast",
    "uzip_alltoall", "uzip_comm_error_detail", "uzip_staged_workspace_bytes", "uzip_compress_staged",
    "uzip_nvls_supported", "uzip_nvls_selftest", "uzip_comm_trace",
]


class UzipError(RuntimeError):
    def __init__(self, status: int, where: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}")
        self.status = status


class CodecParams(ctypes.Structure):
    _fields_ = [("block_symbols", ctypes.c_uint32), ("chunk_blocks", ctypes.c_uint32),
                ("sample_symbols", ctypes.c_uint32), ("global_table", ctypes.c_uint32)]


class Config(ctypes.Structure):
    _fields_ = [("min_compress_bytes", ctypes.c_uint64), ("staging_bytes", ctypes.c_uint64),
                ("pipe_chunk_bytes", ctypes.c_uint64), ("max_ctas", ctypes.c_uint32),
                ("poll_timeout_ms", ctypes.c_uint32), ("codec", CodecParams)]


class Stats(ctypes.Structure):
    _fields_ = [("raw_bytes", ctypes.c_uint64), ("wire_bytes", ctypes.c_uint64),
                ("compressed", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


ALLGATHER_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)

_lib = None
_lib_lock = threading.Lock()


def build(force: bool = False) -> str:
    return _build.build(force=force)


def lib() -> ctypes.CDLL:
    """Load libuzip.so (raises if it has not been built: there is no fallback)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} missing: run `python -m paper_2604_17172_b200._build` "
                                  "(uzip has no CPU fallback)")
            l = ctypes.CDLL(LIB_PATH)
            vp, sz, i32, u64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64
            pp = ctypes.POINTER(CodecParams)
            l.uzip_compress_bound.argtypes = [sz, i32, pp]
            l.uzip_compress_bound.restype = sz
            l.uzip_workspace_bytes.argtypes = [sz, i32, pp]
            l.uzip_workspace_bytes.restype = sz
            l.uzip_workspace_init.argtypes = [vp, sz, vp]
            l.uzip_compress.argtypes = [vp, sz, i32, vp, sz, vp, vp, sz, pp, vp]
            l.uzip_decompress.argtypes = [vp, sz, vp, sz, i32, vp, vp, sz, vp]
            l.uzip_comm_init.argtypes = [ctypes.POINTER(vp), i32, i32, i32, ALLGATHER_FN, vp,
                                         ctypes.POINTER(Config)]
            l.uzip_comm_init_all.argtypes = [ctypes.POINTER(vp), i32, ctypes.POINTER(i32), ctypes.POINTER(Config)]
            l.uzip_comm_destroy.argtypes = [vp]
            l.uzip_send.argtypes = [vp, sz, i32, i32, vp, vp]
            l.uzip_recv.argtypes = [vp, sz, i32, i32, vp, vp]
            l.uzip_allgather.argtypes = [vp, vp, sz, i32, vp, vp]
            l.uzip_reduce_scatter.argtypes = [vp, vp, sz, i32, i32, vp, vp]
            l.uzip_allreduce.argtypes = [vp, vp, sz, i32, i32, vp, vp]
            l.uzip_comm_get_async_error.argtypes = [vp, ctypes.POINTER(i32)]
            l.uzip_get_stats.argtypes = [vp, ctypes.POINTER(Stats)]
            l.uzip_comm_read_staging.argtypes = [vp, i32, i32, vp, sz]
            l.uzip_broadcast.argtypes = [vp, sz, i32, i32, vp, vp]
            l.uzip_alltoall.argtypes = [vp, vp, sz, i32, vp, vp]
            l.uzip_comm_error_detail.argtypes = [vp, vp]
            if hasattr(l, "uzip_compress_staged"):  # (older builds, loaded as tuning variants, lack these)
                l.uzip_staged_workspace_bytes.argtypes = [sz, i32, pp]
                l.uzip_staged_workspace_bytes.restype = sz
                l.uzip_compress_staged.argtypes = [vp, sz, i32, vp, sz, vp, vp, sz, pp, vp, vp, vp]
            if hasattr(l, "uzip_nvls_supported"):
                l.uzip_nvls_supported.argtypes = [i32, ctypes.POINTER(i32)]
                l.uzip_nvls_selftest.argtypes = [i32, sz]
            if hasattr(l, "uzip_comm_trace"):
                l.uzip_comm_trace.argtypes = [vp, vp, sz, ctypes.POINTER(sz)]
            l.uzip_status_string.argtypes = [i32]
            l.uzip_status_string.restype = ctypes.c_char_p
            l.uzip_version.restype = ctypes.c_char_p
            for name in EXPORTED:
                if not hasattr(l, name):
                    continue
                if name not in ("uzip_compress_bound", "uzip_workspace_bytes", "uzip_status_string", "uzip_version",
                                "uzip_staged_workspace_bytes"):
                    getattr(l, name).restype = i32
            _lib = l
    return _lib


def _check(st: int, where: str):
    if st != OK:
        raise UzipError(st, where)


def _stream(stream) -> ctypes.c_void_p:
    """A torch stream, a raw cudaStream_t / CUstream handle (int), or None (torch's current stream)."""
    if stream is None:
        stream = torch.cuda.current_stream()
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def _params(block_symbols=0, chunk_blocks=0, sample_symbols=0, global_table=False):
    return CodecParams(block_symbols, chunk_blocks, sample_symbols, 1 if global_table else 0)


def uz_dtype(t: torch.dtype) -> int:
    if t not in _TORCH_TO_UZ:
        raise UzipError(ERR_UNSUPPORTED_DTYPE, "dtype")
    return _TORCH_TO_UZ[t]


def torch_dtype(d: int) -> torch.dtype:
    return _UZ_TO_TORCH[d]


# ----------------------------------------------------------------------------- sizing
def compress_bound(count: int, dtype: int, **params) -> int:
    p = _params(**params)
    return lib().uzip_compress_bound(count, dtype, ctypes.byref(p))


def workspace_bytes(count: int, dtype: int, **params) -> int:
    p = _params(**params)
    return lib().uzip_workspace_bytes(count, dtype, ctypes.byref(p))


class Workspace:
    """Zero-initialized device workspace (uzip_workspace_init), grown on demand."""

    def __init__(self, device=None):
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.buf = None

    def get(self, nbytes: int, stream=None) -> torch.Tensor:
        nbytes = max(int(nbytes), 64)
        if self.buf is None or self.buf.numel() < nbytes:
            self.buf = torch.empty(nbytes + (nbytes >> 3), dtype=torch.uint8, device=self.device)
            _check(lib().uzip_workspace_init(ctypes.c_void_p(self.buf.data_ptr()), self.buf.numel(),
                                             _stream(stream)), "uzip_workspace_init")
        return self.buf


_ws_cache: dict = {}


def _workspace(nbytes: int, stream=None) -> torch.Tensor:
    dev = torch.cuda.current_device()
    s = (stream or torch.cuda.current_stream()).cuda_stream
    ws = _ws_cache.get((dev, s))
    if ws is None:
        ws = _ws_cache[(dev, s)] = Workspace(dev)
    return ws.get(nbytes, stream)


# ----------------------------------------------------------------------------- codec
def uzip_compress(in_ptr, count, dtype, out_ptr, out_capacity, d_out_bytes_ptr, ws_ptr, ws_bytes, params,
                  stream_ptr) -> int:
    """Raw C-ABI passthrough (pointers as ints)."""
    return lib().uzip_compress(in_ptr, count, dtype, out_ptr, out_capacity, d_out_bytes_ptr, ws_ptr, ws_bytes,
                               ctypes.byref(params) if params is not None else None, stream_ptr)


def uzip_decompress(in_ptr, in_bytes, out_ptr, count, dtype, d_status_ptr, ws_ptr, ws_bytes, stream_ptr) -> int:
    return lib().uzip_decompress(in_ptr, in_bytes, out_ptr, count, dtype, d_status_ptr, ws_ptr, ws_bytes,
                                 stream_ptr)


def compress(x: torch.Tensor, out: torch.Tensor | None = None, out_bytes: torch.Tensor | None = None,
             stream=None, ws: torch.Tensor | None = None, **params):
    """Compress a contiguous CUDA tensor; returns (stream bytes tensor, device int64 byte count)."""
    if not x.is_cuda or not x.is_contiguous():
        raise UzipError(ERR_INVALID_ARG, "compress: need a contiguous CUDA tensor")
    dt = uz_dtype(x.dtype)
    n = x.numel()
    p = _params(**params)
    cap = lib().uzip_compress_bound(n, dt, ctypes.byref(p))
    if cap == 0:
        raise UzipError(ERR_INVALID_ARG, "compress: unsupported params")
    if out is None:
        out = torch.empty(cap, dtype=torch.uint8, device=x.device)
    if out_bytes is None:
        out_bytes = torch.zeros(1, dtype=torch.int64, device=x.device)
    wsb = lib().uzip_workspace_bytes(n, dt, ctypes.byref(p))
    if ws is None:
        ws = _workspace(wsb, stream)
    st = lib().uzip_compress(ctypes.c_void_p(x.data_ptr() if n else 0), n, dt, ctypes.c_void_p(out.data_ptr()),
                             out.numel(), ctypes.c_void_p(out_bytes.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                             ws.numel(), ctypes.byref(p), _stream(stream))
    _check(st, "uzip_compress")
    return out, out_bytes


def compress_staged(x: torch.Tensor, out: torch.Tensor | None = None, out_bytes: torch.Tensor | None = None,
                    stream=None, ws: torch.Tensor | None = None, res_out: torch.Tensor | None = None,
                    split_done=None, **params):
    """Ablation baseline: the staged Steps 1-3 pipeline (uzip_compress_staged); the stream equals
    compress(x, global_table=True).  split_done: optional torch.cuda.Event recorded after Step 1."""
    dt = uz_dtype(x.dtype)
    n = x.numel()
    params["global_table"] = True
    p = _params(**params)
    cap = lib().uzip_compress_bound(n, dt, ctypes.byref(p))
    if out is None:
        out = torch.empty(cap, dtype=torch.uint8, device=x.device)
    if out_bytes is None:
        out_bytes = torch.zeros(1, dtype=torch.int64, device=x.device)
    if ws is None:
        ws = torch.zeros(lib().uzip_staged_workspace_bytes(n, dt, ctypes.byref(p)), dtype=torch.uint8,
                         device=x.device)
    if split_done is not None:
        split_done.record(torch.cuda.current_stream() if stream is None else stream)  # torch creates it lazily
    ev = ctypes.c_void_p(split_done.cuda_event) if split_done is not None else None
    st = lib().uzip_compress_staged(ctypes.c_void_p(x.data_ptr() if n else 0), n, dt,
                                    ctypes.c_void_p(out.data_ptr()), out.numel(),
                                    ctypes.c_void_p(out_bytes.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                    ws.numel(), ctypes.byref(p),
                                    ctypes.c_void_p(res_out.data_ptr()) if res_out is not None else None, ev,
                                    _stream(stream))
    _check(st, "uzip_compress_staged")
    return out, out_bytes


def decompress(stream_buf: torch.Tensor, count: int, dtype, out: torch.Tensor | None = None,
               status: torch.Tensor | None = None, stream=None, ws: torch.Tensor | None = None,
               in_bytes: int | None = None):
    """Decompress a UZB1 stream held in a CUDA uint8 tensor; returns (tensor, device int32 status)."""
    dt = dtype if isinstance(dtype, int) else uz_dtype(dtype)
    if out is None:
        out = torch.empty(count, dtype=torch_dtype(dt), device=stream_buf.device)
    if status is None:
        status = torch.empty(1, dtype=torch.int32, device=stream_buf.device)
    if ws is None:
        ws = _workspace(64, stream)
    nb = stream_buf.numel() * stream_buf.element_size() if in_bytes is None else in_bytes
    st = lib().uzip_decompress(ctypes.c_void_p(stream_buf.data_ptr()), nb,
                               ctypes.c_void_p(out.data_ptr() if count else 0), count, dt,
                               ctypes.c_void_p(status.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                               _stream(stream))
    _check(st, "uzip_decompress")
    return out, status


def nvls_supported(device: int = 0) -> bool:
    v = ctypes.c_int(0)
    _check(lib().uzip_nvls_supported(device, ctypes.byref(v)), "uzip_nvls_supported")
    return bool(v.value)


def nvls_selftest(device: int = 0, nbytes: int = 4 << 20) -> int:
    """Status of the one-device multicast self-test (OK, NOT_IMPLEMENTED without multicast)."""
    return lib().uzip_nvls_selftest(device, nbytes)


def status_string(st: int) -> str:
    return lib().uzip_status_string(st).decode()


def version() -> str:
    return lib().uzip_version().decode()


# ----------------------------------------------------------------------------- communicator
def make_config(min_compress_bytes=0, staging_bytes=0, pipe_chunk_bytes=0, max_ctas=0, poll_timeout_ms=0,
                block_symbols=0, chunk_blocks=0, sample_symbols=0, global_table=False) -> Config:
    return Config(min_compress_bytes, staging_bytes, pipe_chunk_bytes, max_ctas, poll_timeout_ms,
                  _params(block_symbols, chunk_blocks, sample_symbols, global_table))


def torch_bootstrap(group=None):
    """uzip_allgather_fn over torch.distributed (bootstrap only):
    all-gathers `bytes_per_rank` opaque bytes from every rank in rank order."""
    import torch.distributed as dist

    def cb(send, recv, nbytes, ctx):
        try:
            world = dist.get_world_size(group)
            mine = torch.frombuffer(bytearray(ctypes.string_at(send, nbytes)), dtype=torch.uint8)
            dev = torch.device("cuda", torch.cuda.current_device()) \
                if dist.get_backend(group) == "nccl" else torch.device("cpu")
            parts = [torch.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(world)]
            dist.all_gather(parts, mine.to(dev), group=group)
            blob = torch.cat(parts).cpu().numpy().tobytes()
            ctypes.memmove(recv, blob, len(blob))
            return 0
        except Exception as e:  # pragma: no cover - reported as UZIP_ERR_COMM
            print(f"uzip bootstrap failed: {e}")
            return 1
    return ALLGATHER_FN(cb)


class Comm:
    """One rank's communicator (include/uzip.h uzip_comm_t).  Argument marshalling only."""

    def __init__(self, handle: ctypes.c_void_p, nranks: int, rank: int, device: int, keep=None):
        self.h = handle
        self.nranks, self.rank, self.device = nranks, rank, device
        self._keep = keep

    @classmethod
    def from_group(cls, group=None, device: int | None = None, **cfg) -> "Comm":
        """Multi-process init (one process per GPU); torch.distributed bootstraps the IPC handles."""
        import torch.distributed as dist
        dev = torch.cuda.current_device() if device is None else device
        torch.cuda.set_device(dev)
        cb = torch_bootstrap(group)
        h = ctypes.c_void_p()
        c = make_config(**cfg)
        _check(lib().uzip_comm_init(ctypes.byref(h), dist.get_world_size(group), dist.get_rank(group), dev, cb,
                                    None, ctypes.byref(c)), "uzip_comm_init")
        return cls(h, dist.get_world_size(group), dist.get_rank(group), dev, keep=cb)

    @classmethod
    def init_all(cls, nranks: int, devices=None, **cfg) -> list:
        """Single-process init of nranks communicators; devices may repeat (loopback on one GPU)."""
        devices = list(devices) if devices is not None else [torch.cuda.current_device()] * nranks
        hs = (ctypes.c_void_p * nranks)()
        ds = (ctypes.c_int * nranks)(*devices)
        c = make_config(**cfg)
        _check(lib().uzip_comm_init_all(hs, nranks, ds, ctypes.byref(c)), "uzip_comm_init_all")
        return [cls(ctypes.c_void_p(hs[r]), nranks, r, devices[r]) for r in range(nranks)]

    def destroy(self):
        if self.h:
            _check(lib().uzip_comm_destroy(self.h), "uzip_comm_destroy")
            self.h = None

    def send(self, t: torch.Tensor, peer: int, stream=None):
        _check(lib().uzip_send(ctypes.c_void_p(t.data_ptr()), t.numel(), uz_dtype(t.dtype), peer, self.h,
                               _stream(stream)), "uzip_send")

    def recv(self, t: torch.Tensor, peer: int, stream=None):
        _check(lib().uzip_recv(ctypes.c_void_p(t.data_ptr()), t.numel(), uz_dtype(t.dtype), peer, self.h,
                               _stream(stream)), "uzip_recv")

    def all_gather(self, out: torch.Tensor, inp: torch.Tensor, stream=None):
        _check(lib().uzip_allgather(ctypes.c_void_p(inp.data_ptr()), ctypes.c_void_p(out.data_ptr()), inp.numel(),
                                    uz_dtype(inp.dtype), self.h, _stream(stream)), "uzip_allgather")

    def reduce_scatter(self, out: torch.Tensor, inp: torch.Tensor, stream=None, op: int = SUM):
        _check(lib().uzip_reduce_scatter(ctypes.c_void_p(inp.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                         out.numel(), uz_dtype(inp.dtype), op, self.h, _stream(stream)),
               "uzip_reduce_scatter")

    def all_reduce(self, out: torch.Tensor, inp: torch.Tensor | None = None, stream=None, op: int = SUM):
        inp = out if inp is None else inp
        _check(lib().uzip_allreduce(ctypes.c_void_p(inp.data_ptr()), ctypes.c_void_p(out.data_ptr()), out.numel(),
                                    uz_dtype(out.dtype), op, self.h, _stream(stream)), "uzip_allreduce")

    def all_to_all(self, out: torch.Tensor, inp: torch.Tensor, stream=None):
        """out[i*c:(i+1)*c] <- rank i's inp[me*c:(me+1)*c], c = inp.numel() // nranks."""
        _check(lib().uzip_alltoall(ctypes.c_void_p(inp.data_ptr()), ctypes.c_void_p(out.data_ptr()),
                                   inp.numel() // self.nranks, uz_dtype(inp.dtype), self.h, _stream(stream)),
               "uzip_alltoall")

    def broadcast(self, t: torch.Tensor, root: int, stream=None):
        _check(lib().uzip_broadcast(ctypes.c_void_p(t.data_ptr()), t.numel(), uz_dtype(t.dtype), root, self.h,
                                    _stream(stream)), "uzip_broadcast")

    def async_error(self) -> int:
        e = ctypes.c_int(0)
        _check(lib().uzip_comm_get_async_error(self.h, ctypes.byref(e)), "uzip_comm_get_async_error")
        return e.value

    def error_detail(self) -> list:
        buf = (ctypes.c_uint32 * 16)()
        _check(lib().uzip_comm_error_detail(self.h, buf), "uzip_comm_error_detail")
        return list(buf)

    def trace(self, max_events: int = 1 << 20):
        """Tile trace events (UZIP_TRACE=1 at init): numpy array of (kind, job, tile, t_ns) rows."""
        import numpy as np
        buf = np.zeros(2 * max_events, np.uint64)
        n = ctypes.c_size_t(0)
        _check(lib().uzip_comm_trace(self.h, buf.ctypes.data, max_events, ctypes.byref(n)), "uzip_comm_trace")
        ev = buf[: 2 * n.value].reshape(-1, 2)
        kind = (ev[:, 0] >> np.uint64(60)).astype(np.int64)
        job = ((ev[:, 0] >> np.uint64(56)) & np.uint64(15)).astype(np.int64)
        tile = (ev[:, 0] & np.uint64((1 << 56) - 1)).astype(np.int64)
        return np.stack([kind, job, tile, ev[:, 1].astype(np.int64)], axis=1) if n.value else np.zeros((0, 4), np.int64)

    def stats(self) -> dict:
        s = Stats()
        _check(lib().uzip_get_stats(self.h, ctypes.byref(s)), "uzip_get_stats")
        return {"raw_bytes": s.raw_bytes, "wire_bytes": s.wire_bytes, "compressed": bool(s.compressed)}

    def read_staging(self, src: int, slot: int, nbytes: int) -> bytes:
        buf = ctypes.create_string_buffer(nbytes)
        _check(lib().uzip_comm_read_staging(self.h, src, slot, buf, nbytes), "uzip_comm_read_staging")
        return buf.raw
