"""Row sharding + all-gather logic at world_size 2 (and 3) on CPU with gloo.

Each rank computes its row shard with the C oracle (test infrastructure) and
the shards are joined by paper_2512_17970_b200.dist.gather_rows -- the same
code the NCCL path runs on the GPU box.  The joined output must equal the
unsharded oracle output bit for bit (per-row arithmetic is row-independent).
"""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2512_17970_b200.dist import ShardedLayer, shard_bounds


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, rows, cols, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2512_17970_b200 as cg
        from oracle import c_oracle
        from oracle import codegemm_oracle as orc

        q = cg.random_layer(rows, cols, cg.QuantConfig(v=4, m=1, b=8, g=128), seed=5)
        x16 = orc.bench_input_array(cols, 3, 1)
        r0, r1, _ = shard_bounds(rows, world, rank)
        codes = [np.ascontiguousarray(p.codes[r0:r1]) for p in q.planes]
        scales = np.ascontiguousarray(q.scales.scales[r0:r1])
        books = [b.entries for b in q.books]

        def local_fn(x):
            if r1 <= r0:
                return torch.zeros((0, x.shape[1]))
            y = c_oracle.codegemm(codes, books, scales, x.numpy().astype(np.float16), 4, 128)
            return torch.from_numpy(y)

        layer = ShardedLayer(q, rank, world, local_fn=local_fn)
        y = layer(torch.from_numpy(x16))
        if rank == 0:
            np.save(os.path.join(out_dir, "y.npy"), y.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,rows", [(2, 1000), (2, 33), (3, 100), (2, 1)])
def test_sharded_gather_matches_unsharded(world, rows):
    import paper_2512_17970_b200 as cg
    from oracle import c_oracle
    from oracle import codegemm_oracle as orc

    cols = 512
    with tempfile.TemporaryDirectory() as tmp:
        mp.spawn(_worker, args=(world, _free_port(), rows, cols, tmp), nprocs=world, join=True)
        y = np.load(os.path.join(tmp, "y.npy"))
    q = cg.random_layer(rows, cols, cg.QuantConfig(v=4, m=1, b=8, g=128), seed=5)
    x16 = orc.bench_input_array(cols, 3, 1)
    ref = c_oracle.codegemm([p.codes for p in q.planes], [b.entries for b in q.books],
                            q.scales.scales, x16, 4, 128)
    assert y.shape == ref.shape
    assert np.array_equal(y.view(np.uint32), ref.view(np.uint32))


def test_shard_bounds_cover_rows_exactly():
    for rows in (1, 7, 16, 1000, 28672):
        for world in (1, 2, 3, 4, 8):
            got = []
            for rank in range(world):
                r0, r1, per = shard_bounds(rows, world, rank)
                assert 0 <= r0 <= r1 <= rows and r1 - r0 <= per
                got.extend(range(r0, r1))
            assert got == list(range(rows))


def test_gathered_layout_shards_cover_rows_aligned():
    """Exchange buffer layout (dist.GatheredLayout): every layer's gathered
    output at a 256-byte aligned offset; rank shards are whole 16-row groups,
    contiguous, disjoint and cover the rows; each rank's slice starts 16-byte
    aligned (the kernel's vector stores and bulk reduce-adds)."""
    from paper_2512_17970_b200.dist import GatheredLayout, shard_bounds

    rows = [4096, 1024, 1000, 14336, 48]
    for world in (1, 2, 3, 4, 8):
        for n in (1, 3):
            lay = GatheredLayout(rows, n, world)
            assert lay.nbytes >= sum(r * n * 4 for r in rows)
            for i, r in enumerate(rows):
                assert lay.offset[i] % 256 == 0
                if i:
                    assert lay.offset[i] >= lay.offset[i - 1] + rows[i - 1] * n * 4
                covered = 0
                for rank in range(world):
                    r0, r1 = lay.bounds(i, rank)
                    assert r0 == min(r, covered) and r0 <= r1 <= r
                    if r1 > r0:
                        assert r0 % 16 == 0
                        assert (lay.offset[i] + r0 * n * 4) % 16 == 0
                    covered = r1
                assert covered == r
    assert shard_bounds(100, 3, 1) == (34, 68, 34)
    assert shard_bounds(100, 3, 1, align=16) == (48, 96, 48)
