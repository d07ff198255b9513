"""CPU oracle for the Uzip codec and collectives -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this package.  The
product path (``paper_2604_17172_b200``) never imports it and shares no code
with it: the C source ``oracle/uzip_oracle.c`` is a plain single-threaded
restatement of PAPER.md (arxiv 2604.17172) §2.1.2, §3.3
 and §3.4 with the readings listed in DESIGN.md.

Every function is pinned by tests/test_oracle_*.py and tests/test_golden.py
(see DESIGN.md "The oracle and its pins").  The UZB1 byte layout is this
reproduction's definition: the paper publishes no
format or worked stream (P:168 only says the blocks are "merged into a
single contiguous output buffer"), so streams are compared GPU vs oracle.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "uzip_oracle.c")
_HDR = os.path.join(_HERE, "uzip_oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

BF16, F16, F32, E4M3, E5M2 = 0, 1, 2, 3, 4
OK, ERR_INVALID_ARG, ERR_UNSUPPORTED_DTYPE, ERR_CAPACITY, ERR_CORRUPT_STREAM, ERR_SIZE_MISMATCH = range(6)
M = 4096
L = 1 << 15
LANES = 32
RAW_BLOCK = 0xFFFFFFFF
HEADER_BYTES = 64

ELEM_BYTES = {BF16: 2, F16: 2, F32: 4, E4M3: 1, E5M2: 1}
NP_UINT = {BF16: np.uint16, F16: np.uint16, F32: np.uint32, E4M3: np.uint8, E5M2: np.uint8}
GROUP_ELEMS = {BF16: 1, F16: 1, F32: 1, E4M3: 2, E5M2: 1}  # elements per symbol (P:485 e4m3 pairs)
RES_BYTES = {BF16: 1, F16: 1, F32: 3, E4M3: 1, E5M2: 0}    # residual bytes per symbol


def build(force: bool = False) -> str:
    """Compile oracle/liboracle.so with gcc (plain -O2: no fast-math, no FTZ)."""
    with _lock:
        stale = force or not os.path.exists(_LIB) or max(
            os.path.getmtime(_SRC), os.path.getmtime(_HDR)) > os.path.getmtime(_LIB)
        if stale:
            tmp = _LIB + f".tmp{os.getpid()}"
            subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off",
                                   "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


class Params(ctypes.Structure):
    _fields_ = [("block_symbols", ctypes.c_uint32), ("chunk_blocks", ctypes.c_uint32),
                ("sample_symbols", ctypes.c_uint32), ("global_table", ctypes.c_uint32)]


def lib():
    global _lib
    if _lib is None:
        build()
        l = ctypes.CDLL(_LIB)
        vp, sz, u32, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_uint32, ctypes.c_int
        l.uzo_elem_bytes.restype = sz
        l.uzo_split_array.argtypes = [i32, vp, sz, vp, vp]
        l.uzo_join_array.argtypes = [i32, vp, vp, sz, vp]
        l.uzo_histogram.argtypes = [vp, sz, sz, vp]
        l.uzo_normalize.argtypes = [vp, vp]
        l.uzo_encode_block.argtypes = [vp, u32, vp, vp, vp]
        l.uzo_encode_block.restype = u32
        l.uzo_encode_block_l.argtypes = [vp, u32, vp, vp, vp, u32]
        l.uzo_encode_block_l.restype = u32
        l.uzo_decode_block.argtypes = [vp, vp, u32, u32, vp, vp]
        l.uzo_decode_block.restype = i32
        l.uzo_compress_bound.argtypes = [sz, i32, ctypes.POINTER(Params)]
        l.uzo_compress_bound.restype = sz
        l.uzo_compress.argtypes = [i32, vp, sz, ctypes.POINTER(Params), vp, sz, ctypes.POINTER(sz)]
        l.uzo_compress.restype = i32
        l.uzo_decompress.argtypes = [vp, sz, vp, sz, i32]
        l.uzo_decompress.restype = i32
        l.uzo_reduce_sum.argtypes = [i32, ctypes.POINTER(vp), i32, sz, vp]
        l.uzo_reduce.argtypes = [i32, i32, ctypes.POINTER(vp), i32, sz, vp]
        l.uzo_round_from_f32.argtypes = [i32, ctypes.c_float]
        l.uzo_round_from_f32.restype = u32
        l.uzo_widen_to_f32.argtypes = [i32, u32]
        l.uzo_widen_to_f32.restype = ctypes.c_float
        _lib = l
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _params(block_symbols=0, chunk_blocks=0, sample_symbols=0, global_table=False):
    return Params(block_symbols, chunk_blocks, sample_symbols, 1 if global_table else 0)


def as_bits(x: np.ndarray, dtype: int) -> np.ndarray:
    """View raw element bits (uint16 / uint32) of an array or bytes."""
    return np.ascontiguousarray(x).view(NP_UINT[dtype]).reshape(-1)


# ---------------------------------------------------------------- a1 split / join
def split(dtype: int, bits: np.ndarray):
    """Elements -> (symbols, residuals), one per symbol group (e4m3: pairs; len(bits) must be even)."""
    bits = np.ascontiguousarray(bits, dtype=NP_UINT[dtype])
    ge = GROUP_ELEMS[dtype]
    assert bits.size % ge == 0
    n = bits.size // ge
    sym = np.empty(n, np.uint8)
    res = np.empty(n, np.uint32)
    lib().uzo_split_array(dtype, _ptr(bits), n, _ptr(sym), _ptr(res))
    return sym, res


def join(dtype: int, sym: np.ndarray, res: np.ndarray) -> np.ndarray:
    sym = np.ascontiguousarray(sym, dtype=np.uint8)
    res = np.ascontiguousarray(res, dtype=np.uint32)
    out = np.empty(sym.size * GROUP_ELEMS[dtype], NP_UINT[dtype])
    lib().uzo_join_array(dtype, _ptr(sym), _ptr(res), sym.size, _ptr(out))
    return out


# ---------------------------------------------------------------- a2 / a3 tables
def histogram(sym: np.ndarray, limit: int = 0) -> np.ndarray:
    sym = np.ascontiguousarray(sym, dtype=np.uint8)
    cnt = np.zeros(256, np.uint32)
    lib().uzo_histogram(_ptr(sym), sym.size, limit, _ptr(cnt))
    return cnt


def normalize(cnt) -> np.ndarray:
    cnt = np.ascontiguousarray(cnt, dtype=np.uint32)
    f = np.zeros(256, np.uint16)
    lib().uzo_normalize(_ptr(cnt), _ptr(f))
    return f


# ---------------------------------------------------------------- a4 / a8 block codec
def encode_block(sym: np.ndarray, freq: np.ndarray):
    sym = np.ascontiguousarray(sym, dtype=np.uint8)
    freq = np.ascontiguousarray(freq, dtype=np.uint16)
    B = sym.size
    states = np.zeros(32, np.uint32)
    words = np.zeros(max(B, 1), np.uint16)
    K = lib().uzo_encode_block(_ptr(sym), B, _ptr(freq), _ptr(states), _ptr(words))
    return states, words[:K].copy()


def encode_block_l(sym: np.ndarray, freq: np.ndarray, lbits: int):
    """encode_block with the state interval [2^lbits, 2^(lbits+16)) -- 15 is the format (R4), 16 the
    survey prototype's interval (its g1 micro-vector pins the coder)."""
    sym = np.ascontiguousarray(sym, dtype=np.uint8)
    freq = np.ascontiguousarray(freq, dtype=np.uint16)
    B = sym.size
    states = np.zeros(32, np.uint32)
    words = np.zeros(max(B, 1), np.uint16)
    K = lib().uzo_encode_block_l(_ptr(sym), B, _ptr(freq), _ptr(states), _ptr(words), lbits)
    return states, words[:K].copy()


def decode_block(states, words, B: int, freq):
    states = np.ascontiguousarray(states, dtype=np.uint32)
    words = np.ascontiguousarray(words, dtype=np.uint16)
    freq = np.ascontiguousarray(freq, dtype=np.uint16)
    out = np.zeros(B, np.uint8)
    w = words if words.size else np.zeros(1, np.uint16)
    st = lib().uzo_decode_block(_ptr(states), _ptr(w), words.size, B, _ptr(freq), _ptr(out))
    return st, out


def block_bytes(states, words) -> bytes:
    """Serialized coded block (R4): 32 x u32 LE states, K x u16 LE words, zero pad to 16."""
    raw = np.asarray(states, np.uint32).astype("<u4").tobytes() + np.asarray(words, np.uint16).astype("<u2").tobytes()
    return raw + b"\0" * ((-len(raw)) % 16)


# ---------------------------------------------------------------- stream
def compress_bound(n: int, dtype: int, **params) -> int:
    p = _params(**params)
    return lib().uzo_compress_bound(n, dtype, ctypes.byref(p))


def compress(dtype: int, bits: np.ndarray, **params) -> bytes:
    bits = np.ascontiguousarray(bits, dtype=NP_UINT[dtype]).reshape(-1)
    n = bits.size
    p = _params(**params)
    cap = lib().uzo_compress_bound(n, dtype, ctypes.byref(p))
    out = np.zeros(max(cap, 1), np.uint8)
    nbytes = ctypes.c_size_t(0)
    src = bits if n else np.zeros(1, NP_UINT[dtype])
    st = lib().uzo_compress(dtype, _ptr(src), n, ctypes.byref(p), _ptr(out), cap, ctypes.byref(nbytes))
    if st != OK:
        raise RuntimeError(f"oracle compress failed: status {st}")
    return out[: nbytes.value].tobytes()


def decompress(stream: bytes, n: int, dtype: int):
    """Returns (status, bits ndarray)."""
    buf = np.frombuffer(stream, np.uint8).copy() if len(stream) else np.zeros(1, np.uint8)
    out = np.zeros(max(n, 1), NP_UINT[dtype])
    st = lib().uzo_decompress(_ptr(buf), len(stream), _ptr(out), n, dtype)
    return st, out[:n]


def parse_header(stream: bytes) -> dict:
    h = np.frombuffer(stream[:64], np.uint8)
    u32 = lambda o: int(np.frombuffer(stream[o:o + 4], "<u4")[0])
    u64 = lambda o: int(np.frombuffer(stream[o:o + 8], "<u8")[0])
    return dict(magic=bytes(stream[:4]), version=int(np.frombuffer(stream[4:6], "<u2")[0]), dtype=int(h[6]),
                flags=int(h[7]), n=u64(8), B=u32(16), CB=u32(20), S=u32(24), P=int(h[28]), W=int(h[29]),
                Lbits=int(h[30]), n_blocks=u32(32), n_chunks=u32(36), payload_bytes=u64(40), total_bytes=u64(48))


def sections(stream: bytes) -> dict:
    """Section offsets of a UZB1 stream, recomputed from its header (R-Format)."""
    hd = parse_header(stream)
    r16 = lambda v: (v + 15) & ~15
    nb, nc, B = hd["n_blocks"], hd["n_chunks"], hd["B"]
    ncoded = nb * B
    off_res0 = 64
    if hd["dtype"] == F32:
        off_res1 = off_res0 + 2 * ncoded
        off_tab = r16(off_res1 + ncoded)
    else:
        off_res1 = off_res0
        off_tab = r16(off_res0 + RES_BYTES[hd["dtype"]] * ncoded)
    off_coff = off_tab + 512 * nc
    off_dir = r16(off_coff + 8 * nc)
    off_pay = r16(off_dir + 4 * nb)
    off_tail = r16(off_pay + hd["payload_bytes"])
    return dict(hd, off_res0=off_res0, off_res1=off_res1, off_tab=off_tab, off_coff=off_coff,
                off_dir=off_dir, off_pay=off_pay, off_tail=off_tail)


# ---------------------------------------------------------------- a9 fold
SUM, MIN, MAX = 0, 1, 2


def reduce(dtype: int, inputs, op: int = 0) -> np.ndarray:
    """Fold R with op (R11 sum; R25 min/max), rank order."""
    arrs = [np.ascontiguousarray(a, dtype=NP_UINT[dtype]).reshape(-1) for a in inputs]
    n = arrs[0].size
    ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    out = np.zeros(max(n, 1), NP_UINT[dtype])
    lib().uzo_reduce(dtype, op, ptrs, len(arrs), n, _ptr(out))
    return out[:n]


def reduce_sum(dtype: int, inputs) -> np.ndarray:
    arrs = [np.ascontiguousarray(a, dtype=NP_UINT[dtype]).reshape(-1) for a in inputs]
    n = arrs[0].size
    ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    out = np.zeros(max(n, 1), NP_UINT[dtype])
    lib().uzo_reduce_sum(dtype, ptrs, len(arrs), n, _ptr(out))
    return out[:n]


def round_from_f32(dtype: int, v: float) -> int:
    return lib().uzo_round_from_f32(dtype, v)


def widen_to_f32(dtype: int, bits: int) -> float:
    return lib().uzo_widen_to_f32(dtype, bits)


def allgather(dtype: int, inputs):
    """AllGather plain definition: out[r*n+i] = in_r[i] on every rank."""
    return np.concatenate([np.asarray(a, NP_UINT[dtype]).reshape(-1) for a in inputs])


def reduce_scatter(dtype: int, inputs, nranks: int, op: int = 0):
    """ReduceScatter: rank r gets R over shard r of every input."""
    n = np.asarray(inputs[0]).size // nranks
    return [reduce(dtype, [np.asarray(a).reshape(-1)[r * n:(r + 1) * n] for a in inputs], op) for r in range(nranks)]


def allreduce(dtype: int, inputs, op: int = 0):
    return reduce(dtype, inputs, op)


# ---------------------------------------------------------------- O13 wire streams
TILE_BLOCKS = 8  # blocks per tile of the GPU encoder (DESIGN R18); R26 samples one tile


def wire_streams(kind: str, dtype: int, inputs, op: int = 0, **params):
    """Which UZB1 streams a compressed single-round collective puts on the wire:
    a list of (src, dst, phase, stream bytes).  Composed only of compress() and reduce() above.

    p2p:        inputs = [x]: (0, 1, "p2p", compress(x)).
    allgather:  the stream of in_r, sent to every peer.
    reduce_scatter: for each j != r the stream of shard j of in_r, to rank j.
    allreduce:  reduce_scatter's streams ("rs"), then the stream of rank j's reduced shard out_j to
                every peer ("ag").  R26: the allgather phase is coded in the same pass
                as the reduction, so each chunk's table is sampled from the chunk's first tile
                (sample_symbols = 8 B) -- P:364's "first ... of each chunk", read at tile size.
    """
    N = len(inputs)
    xs = [np.ascontiguousarray(a, dtype=NP_UINT[dtype]).reshape(-1) for a in inputs]
    out = []
    if kind == "p2p":
        return [(0, 1, "p2p", compress(dtype, xs[0], **params))]
    if kind == "allgather":
        for r in range(N):
            s = compress(dtype, xs[r], **params)
            out += [(r, d, "ag", s) for d in range(N) if d != r]
        return out
    m = xs[0].size // N
    for r in range(N):
        for j in range(N):
            if j != r:
                out.append((r, j, "rs", compress(dtype, xs[r][j * m:(j + 1) * m], **params)))
    if kind == "reduce_scatter":
        return out
    if kind != "allreduce":
        raise ValueError(kind)
    red = reduce(dtype, xs, op)
    B = params.get("block_symbols") or 4096
    agp = dict(params, sample_symbols=TILE_BLOCKS * B)
    for j in range(N):
        s = compress(dtype, red[j * m:(j + 1) * m], **agp)
        out += [(j, d, "ag", s) for d in range(N) if d != j]
    return out
