"""Bench shapes and engine dispatch (the reference harness's plugin point).

Mirrors ``/root/reference/pkg/src/codegemm/bench.py``: the decoder-block
suites (bench.py:63-74), ``ShapeSpec`` (bench.py:77-85), the seeded inputs
``bench_input`` / ``bench_layer`` (bench.py:162-170) and ``run_engine``
(bench.py:173-189).  ``run_engine`` is a superset on the GPU side:
``"codegemm"`` and ``"codegemm-b200"`` run the fused kernel,
``"codegemm-strict"`` the bit-exact kernel.  The reference's CPU baselines
("dense", "dequant", "dequant-mirrored") are not part of the B200 path.
"""

from __future__ import annotations

import time
from dataclasses import dataclass
from statistics import median

import numpy as np

from .engines import TileConfig, codegemm_gemm
from .errors import ConfigError
from .quantizer import random_layer
from .tensors import Matrix

ENGINES = ("codegemm", "codegemm-b200", "codegemm-strict")

# (name, out_features, in_features, multiplicity per decoder block)
SUITES = {
    "llama8b": (
        ("attn_proj", 4096, 4096, 4),
        ("mlp_gate_up", 14336, 4096, 2),
        ("mlp_down", 4096, 14336, 1),
    ),
    "llama70b": (
        ("attn_proj", 8192, 8192, 4),
        ("mlp_gate_up", 28672, 8192, 2),
        ("mlp_down", 8192, 28672, 1),
    ),
}

# Real Llama-3 GQA projections, reported beside
# the reference suite: fused qkv and the k/v projections.
GQA_SHAPES = {
    "llama8b": (("qkv_fused", 6144, 4096), ("kv_proj", 1024, 4096)),
    "llama70b": (("qkv_fused", 10240, 8192), ("kv_proj", 1024, 8192)),
}


@dataclass(frozen=True)
class ShapeSpec:
    m_batch: int
    n_out: int
    k_in: int
    multiplicity: int = 1
    name: str = ""


def suite_shapes(suite: str, batches=(1,)) -> list:
    if suite not in SUITES:
        raise ConfigError(f"unknown suite {suite!r}")
    return [ShapeSpec(mb, n, k, mult, name) for mb in batches for (name, n, k, mult) in SUITES[suite]]


def bench_input(shape: ShapeSpec, seed: int) -> Matrix:
    rng = np.random.default_rng((seed, shape.k_in, shape.m_batch, 0x1A))
    return Matrix.from_array(rng.standard_normal((shape.k_in, shape.m_batch)))


def bench_layer(shape: ShapeSpec, cfg, seed: int):
    return random_layer(shape.n_out, shape.k_in, cfg, seed=seed ^ shape.n_out ^ shape.k_in)


def run_engine(engine: str, layer, x, tiles: TileConfig, threads: int):
    if engine in ("codegemm", "codegemm-b200"):
        return codegemm_gemm(layer, x, tiles, threads=threads, mode="auto")
    if engine == "codegemm-strict":
        return codegemm_gemm(layer, x, tiles, threads=threads, mode="strict")
    raise ConfigError(f"unknown engine {engine!r} (choose from {', '.join(ENGINES)})")


def time_engine(engine, layer, x, tiles, threads, repeats: int, warmup: int):
    """The reference timing protocol (bench.py:192-214), wall clock in us."""
    if repeats < 1:
        raise ConfigError(f"repeats must be >= 1, got {repeats}")
    if warmup < 0:
        raise ConfigError(f"warmup must be >= 0, got {warmup}")
    counters = None
    for _ in range(warmup):
        _, counters = run_engine(engine, layer, x, tiles, threads)
    samples = []
    for _ in range(repeats):
        t0 = time.perf_counter_ns()
        _, counters = run_engine(engine, layer, x, tiles, threads)
        samples.append((time.perf_counter_ns() - t0) / 1000.0)
    return round(median(samples), 3), round(min(samples), 3), counters
