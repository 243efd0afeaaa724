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

Two ways to join the slices:

* ``ShardedLayer`` / ``gather_rows``: the layer's launch, then NCCL
  ``all_gather_into_tensor``.
* ``PeerExchange`` (cg_comm, include/codegemm_b200.h): the all-gather fused
  into the staged kernel.  Each rank's gathered buffers live in
  one device region that every peer maps (CUDA IPC); after a stage the kernel
  stores its rows straight into every peer's copy over NVLink and releases a
  counter, and the next stage -- in the same launch -- reads the gathered x
  once every rank arrived.  A whole row-sharded decoder block is then ONE
  launch per rank with no collective call.
"""

from __future__ import annotations

import ctypes
import math

import torch
import torch.distributed as dist

from . import _lib
from .errors import ShapeError

XCHG_PUSH = 1  # CG_XCHG_PUSH: y is this rank's rows inside the comm buffer
XCHG_WAIT = 2  # CG_XCHG_WAIT: x was gathered by an earlier launch
IPC_HANDLE_BYTES = 64


def shard_bounds(rows: int, world: int, rank: int, align: int = 1) -> tuple[int, int, int]:
    """(r0, r1, rows_per_rank): equal padded shards so all-gather is uniform.

    ``align`` rounds the shard size up to a multiple (16: whole row groups,
    16-byte aligned slices -- what the exchange path uses)."""
    per = math.ceil(rows / world)
    per = math.ceil(per / align) * align
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


class _DeviceArray:
    """A zero-copy float32 view of comm memory for torch.as_tensor (keeps the comm alive)."""

    def __init__(self, owner, ptr: int, shape):
        self._owner = owner
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4",
                                         "data": (ptr, False), "version": 3, "strides": None}


class PeerExchange:
    """This rank's row-shard exchange region (cg_comm_*).

    ``nbytes`` of gathered buffers (same on every rank); ``ctas`` CTAs per
    launch (0 = every SM; ranks sharing one GPU in tests split the SMs);
    ``timeout_ms`` traps a kernel whose peers never arrive (0 = wait forever).
    Link the ranks with ``connect`` (one process per GPU: IPC handles through
    ``torch.distributed.all_gather_object``) or ``link`` (ranks of one process).
    Every rank must then issue the same sequence of exchange launches.
    """

    def __init__(self, world: int, rank: int, nbytes: int, *, ctas: int = 0,
                 timeout_ms: int = 0, device=None):
        lib = _lib.load()
        dev = torch.cuda.current_device() if device is None else int(device)
        h = ctypes.c_void_p()
        _lib.check(lib.cg_comm_create(world, rank, int(nbytes), ctas, timeout_ms, dev,
                                      ctypes.byref(h)))
        self.handle = h
        self.world, self.rank, self.device, self.nbytes = world, rank, dev, int(nbytes)
        b = ctypes.c_void_p()
        _lib.check(lib.cg_comm_buffer(h, ctypes.byref(b)))
        self.base = int(b.value)

    def view(self, offset: int, rows: int, n: int) -> torch.Tensor:
        """(rows, n) float32 CUDA tensor at byte ``offset`` of the gathered buffers."""
        if offset < 0 or offset % 16 or offset + rows * n * 4 > self.nbytes:
            raise ShapeError(f"view [{offset}, +{rows * n * 4}) outside the {self.nbytes}-byte "
                             "comm buffer or not 16-byte aligned")
        return torch.as_tensor(_DeviceArray(self, self.base + offset, (rows, n)),
                               device=f"cuda:{self.device}")

    def ipc_handle(self) -> bytes:
        buf = ctypes.create_string_buffer(IPC_HANDLE_BYTES)
        _lib.check(_lib.load().cg_comm_ipc_handle(self.handle, buf))
        return buf.raw

    def open_peers(self, handles) -> None:
        if len(handles) != self.world or any(len(h) != IPC_HANDLE_BYTES for h in handles):
            raise ShapeError(f"need {self.world} handles of {IPC_HANDLE_BYTES} bytes")
        blob = b"".join(handles)
        _lib.check(_lib.load().cg_comm_open_peers(self.handle, blob))

    def connect(self, group=None) -> None:
        """Exchange IPC handles over the process group and map every peer's region."""
        handles = [None] * self.world
        dist.all_gather_object(handles, self.ipc_handle(), group=group)
        self.open_peers(handles)

    @staticmethod
    def link(comms) -> None:
        """Ranks of one process (tests): comms[r] is rank r."""
        arr = (ctypes.c_void_p * len(comms))(*[c.handle.value for c in comms])
        lib = _lib.load()
        for c in comms:
            _lib.check(lib.cg_comm_set_peers(c.handle, arr))

    def close(self) -> None:
        if getattr(self, "handle", None) is not None and self.handle.value:
            _lib.load().cg_comm_destroy(self.handle)
            self.handle = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GatheredLayout:
    """Byte offsets of the gathered outputs of row-sharded layers in a comm buffer.

    Layer i's gathered (rows_i, n) float32 output starts at ``offset[i]`` on
    every rank; rank r writes rows [r0, r1) of it (``shard_bounds(.., align=16)``),
    and a later layer reads all rows as its x.
    """

    def __init__(self, rows, n: int, world: int):
        self.rows, self.n, self.world = [int(r) for r in rows], int(n), int(world)
        self.offset, off = [], 0
        for r in self.rows:
            self.offset.append(off)
            off += (r * n * 4 + 255) // 256 * 256
        self.nbytes = off

    def bounds(self, i: int, rank: int) -> tuple[int, int]:
        r0, r1, _ = shard_bounds(self.rows[i], self.world, rank, align=16)
        return r0, r1

    def gathered(self, comm: PeerExchange, i: int) -> torch.Tensor:
        return comm.view(self.offset[i], self.rows[i], self.n)

    def local(self, comm: PeerExchange, i: int) -> torch.Tensor:
        r0, r1 = self.bounds(i, comm.rank)
        return comm.view(self.offset[i] + r0 * self.n * 4, r1 - r0, self.n)
