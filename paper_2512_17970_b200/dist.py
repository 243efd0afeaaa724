"""Row-sharded CodeGEMM across GPUs with an all-gather of the outputs.

North star (BASELINE.json): Llama-3-70B-shaped layers are partitioned along
the output dimension across the GPUs of one box; each GPU owns its rows'
codes and scales (codebooks and x are replicated) and the per-GPU output
slices are joined with an NCCL all-gather over NVLink.  Row r needs only
codes[:, r, :] and scales[r, :], so shards are independent and -- because a
row's arithmetic in the fused kernel does not depend on which rows share its
CTA (tests/test_parity_gpu.py::test_row_shards_bit_identical_to_full_layer) --
the gathered output is bit-identical to the single-GPU output for the same
tiling.  The reference has no distributed path; its in-process analogue is
the row-block split of engines.py:280-284.

One process per GPU; ``torch.distributed`` provides the plumbing (backend
"nccl" on the box, "gloo" in the CPU tests).
"""

from __future__ import annotations

import math

import torch
import torch.distributed as dist


def shard_bounds(rows: int, world: int, rank: int) -> tuple[int, int, int]:
    """(r0, r1, rows_per_rank): equal padded shards so all-gather is uniform."""
    per = math.ceil(rows / world)
    r0 = min(rows, rank * per)
    r1 = min(rows, r0 + per)
    return r0, r1, per


def gather_rows(y_local: torch.Tensor, per: int, world: int, group=None) -> torch.Tensor:
    """All-gather equal (per, n) slices into (world*per, n), rank-major."""
    n = y_local.shape[1]
    if y_local.shape[0] != per:
        pad = torch.zeros((per, n), dtype=y_local.dtype, device=y_local.device)
        pad[: y_local.shape[0]] = y_local
        y_local = pad
    out = torch.empty((world * per, n), dtype=y_local.dtype, device=y_local.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, y_local.contiguous(), group=group)
    else:  # gloo: list form
        parts = list(out.chunk(world, dim=0))
        dist.all_gather(parts, y_local.contiguous(), group=group)
        out = torch.cat(parts, dim=0)
    return out


class ShardedLayer:
    """This rank's row shard of a quantized layer + the output all-gather.

    ``local_fn`` computes y for the shard from x (default: a DeviceLayer on
    this rank's GPU running the fused kernel).  Tests pass a CPU function to
    exercise the sharding and gather logic under gloo.
    """

    def __init__(self, q, rank: int, world: int, *, group=None, local_fn=None, **layer_kw):
        self.rows, self.cols = int(q.rows), int(q.cols)
        self.rank, self.world, self.group = rank, world, group
        self.r0, self.r1, self.per = shard_bounds(self.rows, world, rank)
        self.device_layer = None
        if local_fn is None and self.r1 > self.r0:
            from .engines import DeviceLayer

            self.device_layer = DeviceLayer(q, row_range=(self.r0, self.r1), **layer_kw)
            local_fn = self.device_layer.gemm
        self.local_fn = local_fn

    def local(self, x: torch.Tensor, y_local: torch.Tensor | None = None) -> torch.Tensor:
        n = x.shape[1]
        if self.r1 <= self.r0:
            return torch.zeros((0, n), dtype=torch.float32, device=x.device)
        if y_local is not None and self.device_layer is not None:
            return self.device_layer.gemm(x, y_local)
        return self.local_fn(x)

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        y_local = self.local(x)
        return gather_rows(y_local, self.per, self.world, self.group)[: self.rows]

    __call__ = forward
