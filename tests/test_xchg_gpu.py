"""Row-shard exchange fused into the staged kernel (cg_gemm_stages_xchg).

The exchange replaces the per-layer NCCL all-gather of the row-sharded path:
each rank's kernel stores its rows into every peer's gathered buffer over
peer memory and the next stage reads the gathered x after every rank arrived.
One GPU is available, so ranks are simulated by several comms of one process
("virtual ranks"): the kernel code path is the same -- peer stores go through
the same address deltas and system-scope counters -- only the memory is local.

Parity: in deterministic mode a row's arithmetic does not depend on which rows
share its task or its GPU (test_row_shards_bit_identical_to_full_layer), so the
gathered outputs must equal the single-GPU staged chain bit for bit.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_2512_17970_b200 as cg  # noqa: E402
from paper_2512_17970_b200 import _lib  # noqa: E402
from paper_2512_17970_b200 import dist as cgd  # noqa: E402
from oracle import c_oracle  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402
from helpers import assert_within_tolerance  # noqa: E402

pytestmark = pytest.mark.gpu
DET = _lib.CG_OPT_DETERMINISTIC
PUSH, WAIT = cgd.XCHG_PUSH, cgd.XCHG_WAIT

# a three-layer chain: x0 (2048) -> A (1024 rows) -> B (2048 rows) -> C (512 rows)
SHAPES = [(1024, 2048), (2048, 1024), (512, 2048)]
CFG = cg.QuantConfig(v=4, m=1, b=8, g=128)


def u32(a):
    return np.ascontiguousarray(a).view(np.uint32)


def _qs():
    return [cg.random_layer(r, c, CFG, seed=700 + i) for i, (r, c) in enumerate(SHAPES)]


def _x0():
    return torch.from_numpy(orc.bench_input_array(2048, 1, 21)).cuda()


def _oracle_check(qs, x0, got, what=""):
    """Each gathered output against the C oracle (the pinned restatement of
    codegemm_gemm) fed the binary16 rounding of the previous gathered output --
    the reference's fp16 boundary (cli.py:136) -- within the fast-mode tolerance."""
    x = x0.cpu().numpy() if hasattr(x0, "cpu") else np.asarray(x0)
    for i, q in enumerate(qs):
        ref = c_oracle.codegemm([p.codes for p in q.planes], [b.entries for b in q.books],
                                q.scales.scales, x.astype(np.float16), 4, 128, threads=8)
        assert_within_tolerance(got[i], ref, f"{what} layer {i} vs oracle")
        x = np.asarray(got[i], dtype=np.float32)


def _single_gpu_chain(qs, x0, flags):
    layers = [cg.DeviceLayer(q, u=2, flags=flags) for q in qs]
    ys = [torch.empty((r, 1), dtype=torch.float32, device="cuda") for r, _ in SHAPES]
    cg.gemm_stages(layers, [x0] + ys[:-1], ys, [0, 1, 2])
    return [y.cpu().numpy() for y in ys]


@pytest.mark.parametrize("det", [True, False])
def test_exchange_world1_chain_matches_staged_chain(det):
    qs, x0 = _qs(), _x0()
    flags = DET if det else 0
    ref = _single_gpu_chain(qs, x0, flags)
    lay = cgd.GatheredLayout([r for r, _ in SHAPES], 1, 1)
    comm = cgd.PeerExchange(1, 0, lay.nbytes, timeout_ms=5000)
    layers = [cg.DeviceLayer(q, u=2, flags=flags) for q in qs]
    ys = [lay.local(comm, i) for i in range(3)]
    xs = [x0, lay.gathered(comm, 0), lay.gathered(comm, 1)]
    for _ in range(3):  # counters carry over launches
        for y in ys:
            y.fill_(float("nan"))
        cg.gemm_stages(layers, xs, ys, [0, 1, 2], xchg=[PUSH] * 3, comm=comm)
        got = [lay.gathered(comm, i).cpu().numpy() for i in range(3)]
        _oracle_check(qs, x0, got, "world 1")
        for i in range(3):
            if det:
                assert np.array_equal(u32(got[i]), u32(ref[i])), i
            else:
                assert_within_tolerance(got[i], ref[i], f"exchange chain layer {i}")


def test_exchange_two_ranks_one_stage_per_launch():
    """Each layer a separate launch per rank, ranks interleaved on one stream:
    pushes at the end of a launch, CG_XCHG_WAIT at the start of the next."""
    qs, x0 = _qs(), _x0()
    ref = _single_gpu_chain(qs, x0, DET)
    world = 2
    lay = cgd.GatheredLayout([r for r, _ in SHAPES], 1, world)
    comms = [cgd.PeerExchange(world, r, lay.nbytes, timeout_ms=5000) for r in range(world)]
    cgd.PeerExchange.link(comms)
    layers = [[cg.DeviceLayer(q, u=2, flags=DET, row_range=lay.bounds(i, r))
               for i, q in enumerate(qs)] for r in range(world)]
    for rep in range(3):
        for c in comms:
            for i in range(3):
                lay.gathered(c, i).fill_(float("nan"))
        torch.cuda.synchronize()
        for i in range(3):
            for r in range(world):
                x = x0 if i == 0 else lay.gathered(comms[r], i - 1)
                cg.gemm_stages([layers[r][i]], [x], [lay.local(comms[r], i)], [0],
                               xchg=[PUSH | (WAIT if i else 0)], comm=comms[r])
        torch.cuda.synchronize()
        for r in range(world):
            got = [lay.gathered(comms[r], i).cpu().numpy() for i in range(3)]
            _oracle_check(qs, x0, got, f"rank {r}")
            for i in range(3):
                assert np.array_equal(u32(got[i]), u32(ref[i])), (rep, r, i)


_CONCURRENT = r"""
import sys, numpy as np, torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2512_17970_b200 as cg
from paper_2512_17970_b200 import _lib, dist as cgd
import test_xchg_gpu as t

world = int(sys.argv[1])
qs, x0 = t._qs(), t._x0()
ref = t._single_gpu_chain(qs, x0, t.DET)
sms = torch.cuda.get_device_properties(0).multi_processor_count
lay = cgd.GatheredLayout([r for r, _ in t.SHAPES], 1, world)
comms = [cgd.PeerExchange(world, r, lay.nbytes, ctas=sms // world, timeout_ms=5000)
         for r in range(world)]
cgd.PeerExchange.link(comms)
layers = [[cg.DeviceLayer(q, u=2, flags=t.DET, row_range=lay.bounds(i, r))
           for i, q in enumerate(qs)] for r in range(world)]
streams = [torch.cuda.Stream() for _ in range(world)]
for rep in range(5):
    torch.cuda.synchronize()
    for r in range(world):  # the whole chain in ONE launch per rank, ranks concurrent
        xs = [x0, lay.gathered(comms[r], 0), lay.gathered(comms[r], 1)]
        ys = [lay.local(comms[r], i) for i in range(3)]
        cg.gemm_stages(layers[r], xs, ys, [0, 1, 2], xchg=[t.PUSH] * 3, comm=comms[r],
                       stream=streams[r])
    torch.cuda.synchronize()
    for r in range(world):
        got = [lay.gathered(comms[r], i).cpu().numpy() for i in range(3)]
        if rep == 0:
            t._oracle_check(qs, x0, got, f"world {world} rank {r}")
        for i in range(3):
            assert np.array_equal(t.u32(got[i]), t.u32(ref[i])), (rep, r, i)
print("OK")
"""


@pytest.mark.parametrize("world", [2, 4])
def test_exchange_concurrent_ranks_one_launch_per_chain(world):
    """`world` ranks on one GPU (sms/world CTAs each), each running the whole
    three-stage chain in one launch on its own stream: stage s+1 waits for
    every rank's pushed rows of stage s.  In a subprocess: a rank that never
    arrives traps its kernel (5 s timeout) instead of poisoning this session."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _CONCURRENT, str(world)], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout[-2000:] + r.stderr[-4000:]


def test_exchange_rejects_bad_arguments():
    qs, x0 = _qs(), _x0()
    lay = cgd.GatheredLayout([r for r, _ in SHAPES], 1, 2)
    comm = cgd.PeerExchange(2, 0, lay.nbytes, timeout_ms=5000)
    dl = cg.DeviceLayer(qs[0], u=2, row_range=lay.bounds(0, 0))
    y = lay.local(comm, 0)
    with pytest.raises(ValueError):  # peers not linked yet
        cg.gemm_stages([dl], [x0], [y], [0], xchg=[PUSH], comm=comm)
    other = cgd.PeerExchange(2, 1, lay.nbytes, timeout_ms=5000)
    cgd.PeerExchange.link([comm, other])
    outside = torch.empty((dl.rows, 1), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):  # pushed y outside the comm buffer
        cg.gemm_stages([dl], [x0], [outside], [0], xchg=[PUSH], comm=comm)
    with pytest.raises(ValueError):  # gathered x must be float32 in the buffer
        cg.gemm_stages([dl], [x0], [y], [0], xchg=[PUSH | WAIT], comm=comm)
    with pytest.raises(cg.ConfigError):
        cg.gemm_stages([dl], [x0], [y], [0], xchg=[PUSH])


_TWO_PROCESSES = r"""
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2512_17970_b200 as cg
from paper_2512_17970_b200 import dist as cgd
import test_xchg_gpu as t

rank, world = int(sys.argv[1]), 2
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=sys.argv[2])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(0)
qs, x0 = t._qs(), t._x0()
ref = t._single_gpu_chain(qs, x0, t.DET)
sms = torch.cuda.get_device_properties(0).multi_processor_count
lay = cgd.GatheredLayout([r for r, _ in t.SHAPES], 1, world)
comm = cgd.PeerExchange(world, rank, lay.nbytes, ctas=sms // world, timeout_ms=20000)
comm.connect()  # 64-byte CUDA IPC handles over the (gloo) process group
layers = [cg.DeviceLayer(q, u=2, flags=t.DET, row_range=lay.bounds(i, rank))
          for i, q in enumerate(qs)]
for rep in range(3):
    for i in range(3):
        x = x0 if i == 0 else lay.gathered(comm, i - 1)
        cg.gemm_stages([layers[i]], [x], [lay.local(comm, i)], [0],
                       xchg=[t.PUSH | (t.WAIT if i else 0)], comm=comm)
    torch.cuda.synchronize()
    dist.barrier()
    got = [lay.gathered(comm, i).cpu().numpy() for i in range(3)]
    if rep == 0:
        t._oracle_check(qs, x0, got, f"process rank {rank}")
    for i in range(3):
        assert np.array_equal(t.u32(got[i]), t.u32(ref[i])), (rep, rank, i)
    dist.barrier()
comm.close()
dist.destroy_process_group()
print("OK", rank)
"""


def test_exchange_two_processes_cuda_ipc():
    """Two processes (one GPU, time-sliced): the regions are mapped with
    cudaIpcOpenMemHandle after a handle exchange over torch.distributed --
    the one-process-per-GPU plumbing -- and each layer is one launch per rank."""
    import socket

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = str(s.getsockname()[1])
    procs = [subprocess.Popen([sys.executable, "-c", _TWO_PROCESSES, str(r), port], cwd=root,
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)
             for r in range(2)]
    outs = []
    for p in procs:
        try:
            outs.append(p.communicate(timeout=600))
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
    for r, (p, (out, err)) in enumerate(zip(procs, outs)):
        assert p.returncode == 0 and f"OK {r}" in out, out[-2000:] + err[-4000:]


def test_exchange_small_grid_caps_rows_per_task():
    """A comm with few CTAs makes the planner ask for large tasks; rows per task
    must stay under the shared-memory cap computed for binary32 staged inputs
    (regression: the cap assumed binary16 x and the launch did not fit)."""
    qs = [cg.random_layer(r, c, CFG, seed=800 + i)
          for i, (r, c) in enumerate([(4096, 2048), (2048, 4096)])]
    x0 = _x0()
    lay = cgd.GatheredLayout([4096, 2048], 1, 1)
    comm = cgd.PeerExchange(1, 0, lay.nbytes, ctas=4, timeout_ms=5000)
    layers = [cg.DeviceLayer(q, u=4, flags=DET) for q in qs]
    ys = [lay.local(comm, i) for i in range(2)]
    cg.gemm_stages(layers, [x0, lay.gathered(comm, 0)], ys, [0, 1], xchg=[PUSH] * 2, comm=comm)
    ref0 = layers[0].gemm(x0)
    ref1 = layers[1].gemm(ref0.half())
    assert np.array_equal(u32(ys[0].cpu().numpy()), u32(ref0.cpu().numpy()))
    assert np.array_equal(u32(ys[1].cpu().numpy()), u32(ref1.cpu().numpy()))
