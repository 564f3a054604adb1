"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic: it only draws random numbers and
names the workload shapes.  Both sides (oracle/ and the CUDA path) receive the values
it produces *as data*.

Input recipe (SURVEY reading C4):
  * MLP weights nn.Linear-like: U(-1/sqrt(fan_in), +1/sqrt(fan_in)), fan_in = d for W_gate,
    W_up and W_head, fan_in = I for W_down (SPEC S:210 uses 1/sqrt(d) for every matrix;
    the fan-in form keeps the MLP output O(1) for I >> d).  Drawn in fp32, rounded RNE
    to the API dtype.
  * Hidden states x ~ N(0, 1) (post-norm MLP input, unit RMS like an RMSNorm output).
  * Final-norm gain ~ U(0.5, 1.5).
  * KV stand-in (attention is out of scope): N(0, 1) values, [S, 2*d_kv].
  * Seeds: layer weights 1234 + layer, hidden 42, head 7, gain 11, kv 100 + layer.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

SEED_W = 1234
SEED_X = 42
SEED_HEAD = 7
SEED_GAIN = 11
SEED_KV = 100
SEED_ROWS = 2024


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config.  L_ext / d_kv are public model configs."""
    name: str
    hidden: int
    intermediate: int
    S: int
    M: int            # number of mini-sequences the config fixes (C = ceil(S/M))
    vocab: int
    layers: int
    d_kv: int
    dtype: str        # "f32" | "bf16"
    eps: float = 1e-5
    minseq_len: int = 0  # explicit C (the paper's chunk 8192); 0 -> C = ceil(S / M)

    @property
    def C(self) -> int:
        return self.minseq_len or (self.S + self.M - 1) // self.M


# BASELINE.json "configs" (index = position in that list).  Configs 3-5 use the paper's chunk
# size C = 8192: M = ceil(S / 8192) = 16 / 19 (tail 7544) / 56 (tail 4440).
CONFIGS = {
    0: Workload("cfg1-f32-d256-I688-S1024-M4-V1000", 256, 688, 1024, 4, 1000, 1, 64, "f32"),
    1: Workload("cfg2-llama3-8b-mlp-S65536-M8", 4096, 14336, 65536, 8, 128256, 32, 1024, "bf16"),
    2: Workload("cfg3-qwen2.5-7b-28L-S131072", 3584, 18944, 131072, 16, 152064, 28, 512, "bf16", 1e-6, 8192),
    3: Workload("cfg4-mistral-nemo-12b-40L-S155000", 5120, 14336, 155000, 19, 131072, 40, 1024, "bf16", 1e-5, 8192),
    4: Workload("cfg5-llama3-8b-32L-S455000", 4096, 14336, 455000, 56, 128256, 32, 1024, "bf16", 1e-5, 8192),
}


def torch_dtype(name: str) -> torch.dtype:
    return {"f32": torch.float32, "bf16": torch.bfloat16}[name]


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def uniform(shape, bound: float, seed: int, device="cpu", dtype=torch.float32) -> torch.Tensor:
    g = _gen(seed, device)
    t = torch.empty(shape, dtype=torch.float32, device=device)
    t.uniform_(-bound, bound, generator=g)
    return t.to(dtype)


def normal(shape, seed: int, device="cpu", dtype=torch.float32, std: float = 1.0) -> torch.Tensor:
    g = _gen(seed, device)
    t = torch.empty(shape, dtype=torch.float32, device=device)
    t.normal_(0.0, std, generator=g)
    return t.to(dtype)


def mlp_weights(d: int, I: int, layer: int = 0, device="cpu", dtype=torch.float32):
    """(W_gate [I,d], W_up [I,d], W_down [d,I]) for one layer, nn.Linear layout."""
    base = SEED_W + 1000 * layer
    wg = uniform((I, d), 1.0 / math.sqrt(d), base + 0, device, dtype)
    wu = uniform((I, d), 1.0 / math.sqrt(d), base + 1, device, dtype)
    wd = uniform((d, I), 1.0 / math.sqrt(I), base + 2, device, dtype)
    return wg, wu, wd


def hidden(S: int, d: int, device="cpu", dtype=torch.float32, seed: int = SEED_X) -> torch.Tensor:
    return normal((S, d), seed, device, dtype)


def head_weight(V: int, d: int, device="cpu", dtype=torch.float32) -> torch.Tensor:
    return uniform((V, d), 1.0 / math.sqrt(d), SEED_HEAD, device, dtype)


def norm_gain(d: int, device="cpu", dtype=torch.float32) -> torch.Tensor:
    g = _gen(SEED_GAIN, device)
    t = torch.empty((d,), dtype=torch.float32, device=device)
    t.uniform_(0.5, 1.5, generator=g)
    return t.to(dtype)


def kv_standin(S: int, d_kv: int, layer: int, device="cpu", dtype=torch.bfloat16) -> torch.Tensor:
    """Stand-in for one layer's K,V ([S, 2*d_kv]); attention itself is out of scope."""
    return normal((S, 2 * d_kv), SEED_KV + layer, device, dtype)


def sample_rows(S: int, C: int, n_random: int = 512, seed: int = SEED_ROWS):
    """Rows for sampled parity: n_random seeded rows, rows 0 and S-1, and both sides of
    every mini-sequence boundary (i*C - 1, i*C).  Sorted, unique."""
    g = _gen(seed, "cpu")
    rnd = torch.randint(0, S, (min(n_random, S),), generator=g).tolist()
    rows = set(rnd) | {0, S - 1}
    for b in range(C, S, C):
        rows.add(b - 1)
        rows.add(b)
    return sorted(r for r in rows if 0 <= r < S)
