"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no split, no table, no coder,
no reduction): it only draws seeded tensors whose shapes and value
distributions follow the paper's workloads:

  W   bf16(N(0, 0.02))          LLM weights        (Table 1 weight; RL sync P:663-669)
  U   bf16(U[-1, 1])            the paper's own synthetic input
  A   [T, 4096] N(0,1) * exp(N(0, 0.5^2)) per channel, channels 7 and 1337 x 64
                                activations        (Table 1 activation)
  KV  [2, 16, 8, 128] vLLM KV blocks; K scaled per dim by exp(N(0, 0.5^2)), V = N(0,1)
                                KV-cache transfer
  G   fp32 N(0, 1e-3)           gradients          (Table 1 gradient)
  edge: zeros, ones, random bits, NaN/Inf/denormal/-0 mixes

All functions return numpy arrays of raw element bits (uint16 for bf16/f16,
uint32 for f32) so both sides read exactly the same bytes.
"""
from __future__ import annotations

import numpy as np
import torch

BF16, F16, F32, E4M3, E5M2 = 0, 1, 2, 3, 4
_TORCH = {BF16: torch.bfloat16, F16: torch.float16, F32: torch.float32, E4M3: torch.float8_e4m3fn,
          E5M2: torch.float8_e5m2}
_UINT = {BF16: np.uint16, F16: np.uint16, F32: np.uint32, E4M3: np.uint8, E5M2: np.uint8}


def _gen(seed: int) -> torch.Generator:
    g = torch.Generator(device="cpu")
    g.manual_seed(int(seed))
    return g


def _bits(t: torch.Tensor, dtype: int) -> np.ndarray:
    t = t.to(_TORCH[dtype]).contiguous()
    if dtype == F32:
        return t.view(torch.int32).numpy().view(np.uint32).reshape(-1).copy()
    if dtype in (E4M3, E5M2):
        return t.view(torch.uint8).numpy().reshape(-1).copy()
    return t.view(torch.int16).numpy().view(np.uint16).reshape(-1).copy()


def normal(n: int, sigma: float, seed: int, dtype: int = BF16) -> np.ndarray:
    """dtype(N(0, sigma)) -- the W recipe for sigma=0.02 (fp32 draw, RNE cast)."""
    return _bits(torch.randn(n, generator=_gen(seed), dtype=torch.float32) * sigma, dtype)


def weights(n: int, seed: int, dtype: int = BF16) -> np.ndarray:
    return normal(n, 0.02, seed, dtype)


def uniform(n: int, seed: int, dtype: int = BF16) -> np.ndarray:
    """dtype(U[-1, 1]) -- the paper's synthetic input."""
    return _bits(torch.rand(n, generator=_gen(seed), dtype=torch.float32) * 2.0 - 1.0, dtype)


def activations(tokens: int, seed: int, hidden: int = 4096, dtype: int = BF16) -> np.ndarray:
    g = _gen(seed)
    scale = torch.exp(torch.randn(hidden, generator=g) * 0.5)
    scale[7] *= 64.0
    if hidden > 1337:
        scale[1337] *= 64.0
    x = torch.randn(tokens, hidden, generator=g) * scale
    return _bits(x, dtype)


def kv_blocks(nblocks: int, seed: int, dtype: int = BF16) -> np.ndarray:
    """Llama-3-8B vLLM KV blocks [nblocks, 2 (K,V), 16 tokens, 8 heads, 128]."""
    g = _gen(seed)
    kscale = torch.exp(torch.randn(8, 128, generator=g) * 0.5)
    k = torch.randn(nblocks, 16, 8, 128, generator=g) * kscale
    v = torch.randn(nblocks, 16, 8, 128, generator=g)
    return _bits(torch.stack([k, v], dim=1), dtype)


def gradients(n: int, seed: int) -> np.ndarray:
    return normal(n, 1e-3, seed, F32)


def random_bits(n: int, seed: int, dtype: int = BF16) -> np.ndarray:
    rng = np.random.default_rng(seed)
    hi = 1 << (32 if dtype == F32 else (8 if dtype in (E4M3, E5M2) else 16))
    return rng.integers(0, hi, size=n, dtype=np.uint64).astype(_UINT[dtype])


def special_mix(n: int, seed: int, dtype: int = BF16) -> np.ndarray:
    """NaN payloads, +-Inf, denormals, +-0 and ordinary values interleaved."""
    rng = np.random.default_rng(seed)
    if dtype == F32:
        pool = np.array([0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0x7F800001,
                         0xFFFFFFFF, 0x00000001, 0x807FFFFF, 0x3F800000, 0xBF800000, 0x7F7FFFFF],
                        np.uint32)
    elif dtype == BF16:
        pool = np.array([0x0000, 0x8000, 0x7F80, 0xFF80, 0x7FC0, 0x7F81, 0xFFFF, 0x0001, 0x807F,
                         0x3F80, 0xBF80, 0x7F7F], np.uint16)
    elif dtype in (E4M3, E5M2):  # zeros, NaN (e4m3fn 0x7F/0xFF), e5m2 +-inf 0x7C/0xFC, denormals, max
        pool = np.array([0x00, 0x80, 0x7F, 0xFF, 0x7C, 0xFC, 0x01, 0x81, 0x7E, 0x38, 0x7B, 0xFB], np.uint8)
    else:
        pool = np.array([0x0000, 0x8000, 0x7C00, 0xFC00, 0x7E00, 0x7C01, 0xFFFF, 0x0001, 0x83FF,
                         0x3C00, 0xBC00, 0x7BFF], np.uint16)
    pick = rng.integers(0, pool.size, size=n)
    out = pool[pick].copy()
    mix = rng.random(n) < 0.3
    out[mix] = random_bits(int(mix.sum()), seed + 1, dtype)
    return out


def constant(n: int, value_bits: int, dtype: int = BF16) -> np.ndarray:
    return np.full(n, value_bits, _UINT[dtype])


def lcg_symbols(n: int, seed: int) -> np.ndarray:
    """SURVEY.md 8(c) micro-vector generator: x0 = seed,
    x_{i+1} = (1664525 x_i + 1013904223) mod 2^32, sym[i] = 0x7E - min(clz32(x_{i+1}), 20)."""
    out = np.empty(n, np.uint8)
    x = seed & 0xFFFFFFFF
    for i in range(n):
        x = (1664525 * x + 1013904223) & 0xFFFFFFFF
        clz = 32 - x.bit_length()
        out[i] = 0x7E - min(clz, 20)
    return out


def torch_dtype(dtype: int):
    return _TORCH[dtype]
