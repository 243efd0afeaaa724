"""Benchmark of the B200 CodeGEMM decode GEMV (driver contract: one JSON line).

Metric (BASELINE.json): "us/layer & HBM GB/s (frac of roofline), 2-bit
Llama-3 8B/70B decode, batch 1".  ``value`` is whole-job HBM throughput in
GB/s: algorithmic bytes (codes at b bits + binary16 scales + binary16
codebooks + x + y) of every layer in one decoder block, divided
by the device time of the block.  Per-layer microseconds are in ``us_per_layer``.

Workloads (a "step" = the linear layers of one decoder block, the
reference's bench suite with its multiplicities, bench.py:63-74):
  8b  (default at N=1) : 4 x 4096x4096, 2 x 14336x4096, 1 x 4096x14336
  70b (default at N>1) : 4 x 8192x8192, 2 x 28672x8192, 1 x 8192x28672, rows
                         sharded over the N GPUs + NCCL all-gather per layer
At N=1 a step is ONE persistent launch of the fused kernel (cg_gemm_stages):
a dependency chain {q,k,v} -> {o} -> {gate,up} -> {down} with grid barriers
between the stages, where o reads y_q, gate/up read y_o and down reads y_gate
(binary32, rounded to binary16 as read) -- real data dependencies, no work
skipped.  At N>1 the 70B block runs row-sharded with grouped launches and an
NCCL all-gather per layer.  Every layer of a step has its own weights; steps
rotate through enough distinct copies of the block that the weight stream is
larger than L2 (inputs larger than L2: no cache flush needed).  Steps are
replayed from CUDA graphs; time is CUDA events on the launching stream, max
over ranks.

``--impl reference`` times the reference's CPU algorithm (the oracle port of
engines.py:245-316, oracle/codegemm_oracle.py) on a bounded sample of the same
workload on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "μs/layer & HBM GB/s (frac of roofline), 2-bit Llama-3 8B/70B decode, batch 1"
L2_BYTES = 126 * 1024 * 1024
CONFIGS = {"m1v4g128": dict(v=4, m=1, b=8, g=128), "m2v8g128": dict(v=8, m=2, b=8, g=128)}
SUITES = {
    "8b": (("attn_proj", 4096, 4096, 4), ("mlp_gate_up", 14336, 4096, 2),
           ("mlp_down", 4096, 14336, 1)),
    "70b": (("attn_proj", 8192, 8192, 4), ("mlp_gate_up", 28672, 8192, 2),
            ("mlp_down", 8192, 28672, 1)),
}


def layer_bytes(rows: int, cols: int, cfg: dict, n: int, with_io: bool = True) -> int:
    """Algorithmic HBM bytes of one layer call."""
    v, m, b, g = cfg["v"], cfg["m"], cfg["b"], cfg["g"]
    codes = (rows * (cols // v) * m * b + 7) // 8
    scales = 2 * rows * (cols // (cols if g == -1 else g))
    books = 2 * m * (1 << b) * v
    io = 2 * cols * n + 4 * rows * n if with_io else 0
    return codes + scales + books + io


# launch groups of a decoder block (indices into block_spec): layers reading
# the same x share one grouped launch -- q,k,v | o | gate,up | down
STEP_GROUPS = ((0, 1, 2), (3,), (4, 5), (6,))
# the staged step (N=1): stage of each layer and the layer whose y it reads
STEP_STAGES = (0, 0, 0, 1, 2, 2, 3)
STEP_XSRC = (None, None, None, 0, 3, 3, 4)
TILING_U = int(os.environ.get("CG_BENCH_U", "0"))  # one tiling for every layer of a staged launch (0: 4 // m)


def block_spec(workload: str):
    return [(name, rows, cols) for (name, rows, cols, mult) in SUITES[workload] for _ in range(mult)]


def make_layer(rows, cols, cfg, seed):
    import paper_2512_17970_b200 as cg

    qc = cg.QuantConfig(v=cfg["v"], m=cfg["m"], b=cfg["b"], g=cfg["g"])
    return cg.random_layer(rows, cols, qc, seed=seed)


def bench_config(args, n: int, world: int) -> dict:
    """The workload dict both arms print (identical, so the driver's same_config holds)."""
    return {"workload": f"llama{args.workload} decoder-block linears (reference suite x "
                        f"multiplicity), {args.config}, batch {n}",
            "config": args.config, "batch": n, "layers_per_step": len(block_spec(args.workload)),
            "parallelism": (f"rows sharded over {world} GPUs" if world > 1 else "single GPU")}


def layer_seed(copy: int, idx: int, rows: int, cols: int) -> int:
    # copy 0, first layer of each shape: the reference's bench_layer seed (bench.py:168-170)
    return (0 ^ rows ^ cols) if copy == 0 and idx == 0 else 1_000_003 * (copy + 1) + 7919 * idx


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled while the timed region runs."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "50", "-f", self.path],
                stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if self.proc is None or not self.path or not os.path.exists(self.path):
            return None
        rows = []
        with open(self.path) as fh:
            for line in fh:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return None

        def num(s):
            try:
                return float(s)
            except ValueError:
                return None

        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# --------------------------------------------------------------------------- CPU
def cpu_baseline(spec, cfg, n, budget_s: float = 20.0):
    """The oracle port (reference algorithm, oracle/codegemm_oracle.py) on host cores."""
    from oracle import c_oracle
    from oracle import codegemm_oracle as orc

    # numpy port: the reference's own vectorisation (engines.py:245-316), 1 thread
    # (its ThreadPool is GIL-bound: threads>1 is slower)
    done_bytes, t_used, layers_done = 0, 0.0, 0
    for idx, (name, rows, cols) in enumerate(spec):
        q = make_layer(rows, cols, cfg, layer_seed(0, idx, rows, cols))
        x = orc.bench_input_array(cols, n, 0)
        codes = [p.codes for p in q.planes]
        books = [b.entries for b in q.books]
        t0 = time.perf_counter()
        orc.codegemm(codes, books, q.scales.scales, x, cfg["v"], cfg["g"], 32, 2048)
        t_used += time.perf_counter() - t0
        done_bytes += layer_bytes(rows, cols, cfg, n)
        layers_done += 1
        if t_used > budget_s:
            break
    port = {"value": round(done_bytes / t_used / 1e9, 4), "unit": "GB/s", "cores": 1,
            "kind": "port",
            "sample": f"{layers_done} layers of one decoder block through the numpy restatement "
                      f"of codegemm_gemm, threads=1 ({t_used:.1f} s)"}
    # C restatement, all host threads (a stronger CPU reference point, same bits)
    threads = os.cpu_count() or 1
    done_bytes, t_used = 0, 0.0
    for idx, (name, rows, cols) in enumerate(spec):
        q = make_layer(rows, cols, cfg, layer_seed(0, idx, rows, cols))
        x = orc.bench_input_array(cols, n, 0)
        t0 = time.perf_counter()
        c_oracle.codegemm([p.codes for p in q.planes], [b.entries for b in q.books],
                          q.scales.scales, x, cfg["v"], cfg["g"], 32, threads)
        t_used += time.perf_counter() - t0
        done_bytes += layer_bytes(rows, cols, cfg, n)
    port_c = {"value": round(done_bytes / t_used / 1e9, 4), "unit": "GB/s", "cores": threads,
              "kind": "port", "sample": "one decoder block through the C restatement "
                                         f"(oracle/cg_oracle.c), {threads} pthreads"}
    return port, port_c


def run_reference(args, spec, cfg, n, rank, world):
    """--impl reference: the reference CPU algorithm (oracle port), rank 0 only."""
    if rank != 0:
        return
    from oracle import codegemm_oracle as orc

    # bounded sample: whole layers for 8B, a row sample of each layer for 70B
    frac = 1 if args.workload == "8b" else 8
    jobs = []
    for idx, (name, rows, cols) in enumerate(spec):
        q = make_layer(rows, cols, cfg, layer_seed(0, idx, rows, cols))
        r = rows // frac
        codes = [np.ascontiguousarray(p.codes[:r]) for p in q.planes]
        jobs.append((codes, [b.entries for b in q.books], np.ascontiguousarray(q.scales.scales[:r]),
                     orc.bench_input_array(cols, n, 0), r, cols))
    step_bytes = sum(layer_bytes(r, c, cfg, n) for (_, _, _, _, r, c) in jobs)

    def step():
        for codes, books, scales, x, r, c in jobs:
            orc.codegemm(codes, books, scales, x, cfg["v"], cfg["g"], 32, 2048)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    value = step_bytes * args.steps / dt / 1e9
    sample = (f"per step: the {len(jobs)} layers of one {args.workload} decoder block"
              + ("" if frac == 1 else f", first 1/{frac} of each layer's rows")
              + " through the numpy restatement of codegemm_gemm (engines.py:245-316), threads=1 "
                "(the reference's ThreadPool is GIL-bound; 1 thread is its fastest setting)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "u8/f16->f32",
        "data": "synthetic (reference generators: random_layer, bench_input)",
        "config": bench_config(args, n, world),
        "setup": "CPU: the numpy restatement of the reference engine (oracle/codegemm_oracle.py), "
                 "same layers and inputs as the GPU arm",
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------- extras
GQA_8B = (("qkv (fused q,k,v GQA)", 6144, 4096), ("o", 4096, 4096), ("gate", 14336, 4096),
          ("up", 14336, 4096), ("down", 4096, 14336))
GQA_STAGES = (0, 1, 2, 2, 3)
GQA_XSRC = (None, 0, 1, 1, 2)


def measure_extras(args, cfg, n, blocks, spec, kern, ref_api_layers, peak, capture, timed, stream,
                   dev):
    """Secondary lines of the N=1 run (SURVEY.md §8d configs 1, 2-GQA, 4 and the
    reference-API end-to-end leg).  Each is device time over CUDA graphs with
    weights rotated over copies larger than L2, except the e2e leg (wall clock)."""
    import torch

    import paper_2512_17970_b200 as cg
    from oracle import codegemm_oracle as orc

    out = {}
    # ---- config 1: one 4096x4096 layer alone (back-to-back launches, rotating copies)
    if "attn_proj" in kern:
        us = kern["attn_proj"][0]
        b1 = layer_bytes(4096, 4096, cfg, n)
        out["config1_layer"] = {"shape": "4096x4096", "us_per_launch": round(us, 3),
                                "GB/s": round(b1 / (us * 1e-6) / 1e9, 1),
                                "frac_of_measured_hbm": round(b1 / (us * 1e-6) / 1e9 / peak, 4),
                                "bytes": b1,
                                "note": "one fused launch per layer: its fixed cost (launch, "
                                        "Psumbook build, split-K flush) is not amortised over a "
                                        "block"}
    # ---- config 2 with the real Llama-3-8B GQA shapes (fused qkv 6144x4096)
    try:
        gq_bytes = sum(layer_bytes(r, c, cfg, n) for _, r, c in GQA_8B)
        gw = sum(layer_bytes(r, c, cfg, n, with_io=False) for _, r, c in GQA_8B)
        gcopies = max(2, -(-3 * L2_BYTES // gw))
        gblocks = []
        for cp in range(gcopies):
            lay = [cg.DeviceLayer(make_layer(r, c, cfg, 77_000 + 100 * cp + i), u=TILING_U)
                   for i, (_, r, c) in enumerate(GQA_8B)]
            x0 = torch.from_numpy(orc.bench_input_array(4096, n, 500 + cp)).to(dev)
            ys = [torch.empty((r, n), dtype=torch.float32, device=dev) for _, r, c in GQA_8B]
            # o reads the q rows of the fused qkv output (the attention output's width)
            xs = [x0 if src is None else (ys[src][:4096] if src == 0 else ys[src])
                  for src in GQA_XSRC]
            gblocks.append(cg.StagedLaunch(lay, xs, ys, list(GQA_STAGES)))
        g = capture(lambda: [b() for b in gblocks])
        timed([g], 3 * gcopies, gcopies)
        reps = 50 * gcopies
        us = timed([g], reps, gcopies) / reps * 1e3
        out["gqa_block"] = {"shapes": [f"{nm} {r}x{c}" for nm, r, c in GQA_8B],
                            "us_per_block": round(us, 3),
                            "GB/s": round(gq_bytes / (us * 1e-6) / 1e9, 1),
                            "frac_of_measured_hbm": round(gq_bytes / (us * 1e-6) / 1e9 / peak, 4),
                            "bytes_per_block": gq_bytes,
                            "launch": "one staged launch per block: {qkv} -> {o} -> {gate,up} "
                                      "-> {down}, real data dependencies; "
                                      f"{gcopies} block copies rotated"}
        del gblocks, g
    except Exception as e:  # (a secondary line never sinks the bench)
        out["gqa_block"] = {"error": repr(e)[:200]}
    # ---- the block's layers as INDEPENDENT layers (the reference bench protocol,
    #      bench.py:192-214: every layer on its own input, no data dependencies),
    #      two blocks (14 layers) per persistent launch in one stage: contiguous
    #      per-CTA task ranges, Psumbook reused across a CTA's tasks of one K-slice
    try:
        if n == 1 and len(blocks) >= 2 and 2 * len(spec) <= 16:
            plans = [cg.StagedLaunch([L["layer"] for L in blocks[j] + blocks[j + 1]],
                                     [L["x"] for L in blocks[j] + blocks[j + 1]],
                                     [L["y"] for L in blocks[j] + blocks[j + 1]],
                                     [0] * (2 * len(spec)))
                     for j in range(0, len(blocks) - 1, 2)]
            g = capture(lambda: [pl() for pl in plans])
            nb = 2 * len(plans)
            timed([g], 3 * nb, nb)
            reps = 50 * nb
            us = timed([g], reps, nb) / reps * 1e3
            ib = sum(layer_bytes(r, c, cfg, n) for _, r, c in spec)
            out["independent_layers"] = {
                "us_per_block": round(us, 3), "GB/s": round(ib / (us * 1e-6) / 1e9, 1),
                "frac_of_measured_hbm": round(ib / (us * 1e-6) / 1e9 / peak, 4),
                "bytes_per_block": ib,
                "launch": "two blocks' 7 layers each on its own input (no data dependencies, "
                          "the reference bench protocol) in one persistent launch, one stage; "
                          f"{len(blocks)} block copies rotated"}
            del plans, g
    except Exception as e:  # (a secondary line never sinks the bench)
        out["independent_layers"] = {"error": repr(e)[:200]}
    # ---- config 4: batch sweep on the 8B block (reference protocol: layers timed
    #      independently, block = sum over the suite with multiplicities); the same
    #      shapes as dense binary16 weights through cuBLAS for comparison
    try:
        sweep = []
        uniq = {}
        for idx, (name, r, c) in enumerate(spec):
            uniq.setdefault(name, (idx, r, c, 0))
            uniq[name] = (uniq[name][0], r, c, uniq[name][3] + 1)
        # (dense: 4 distinct weight copies per shape, > L2 together for every shape)
        dense_w = {name: [torch.randn((r, c), device=dev, dtype=torch.float16) * 0.02
                          for _ in range(4)] for name, (idx, r, c, mult) in uniq.items()}
        for nb in (4, 8, 16, 32):
            per, per_dense = {}, {}
            for name, (idx, r, c, mult) in uniq.items():
                xs = [torch.from_numpy(orc.bench_input_array(c, nb, k)).to(dev)
                      for k in range(len(blocks))]
                ys = [torch.empty((r, nb), dtype=torch.float32, device=dev)
                      for _ in range(len(blocks))]
                lays = [blocks[k][idx]["layer"] for k in range(len(blocks))]
                gk = capture(lambda lays=lays, xs=xs, ys=ys: [l.gemm(x, y) for l, x, y in
                                                               zip(lays, xs, ys)])
                timed([gk], 2)
                rr = 20
                per[name] = timed([gk], rr) / (rr * len(blocks)) * 1e3
                xd = xs[0]
                gd = capture(lambda ws=dense_w[name], xd=xd: [torch.matmul(w, xd) for w in ws])
                timed([gd], 2)
                per_dense[name] = timed([gd], rr) / (rr * 4) * 1e3
                del gk, gd
            blk = sum(per[nm] * m for nm, (i, r, c, m) in uniq.items())
            blk_d = sum(per_dense[nm] * m for nm, (i, r, c, m) in uniq.items())
            byt = sum(layer_bytes(r, c, cfg, nb) * m for nm, (i, r, c, m) in uniq.items())
            sweep.append({"batch": nb, "kernel": "K4 batch (mma.sync, codebook dequantised "
                                                 "in registers)",
                          "us_per_layer": {f"{nm} {r}x{c}": round(per[nm], 2)
                                           for nm, (i, r, c, m) in uniq.items()},
                          "us_per_block": round(blk, 2),
                          "GB/s": round(byt / (blk * 1e-6) / 1e9, 1),
                          "cublas_fp16_dense_us_per_block": round(blk_d, 2),
                          "dense_note": "torch.matmul of binary16 weights (4 copies per shape "
                                        "rotated), the paper's A.4 comparison"})
        out["batch_sweep"] = sweep
        del dense_w
    except Exception as e:
        out["batch_sweep"] = {"error": repr(e)[:200]}
    # ---- end to end the way a reference user calls it: codegemm_gemm(q, Matrix(x))
    #      per layer with numpy buffers (engines.py:245-263; timed like bench.py:192-214)
    try:
        xs_h = [cg.Matrix(orc.bench_input_array(q.cols, n, 900 + i))
                for i, q in enumerate(ref_api_layers)]
        for q, x in zip(ref_api_layers, xs_h):  # warm-up: uploads and prepacks once per layer
            cg.codegemm_gemm(q, x)
        steps = 20
        t0 = time.perf_counter()
        for _ in range(steps):
            for q, x in zip(ref_api_layers, xs_h):
                cg.codegemm_gemm(q, x)
        dt = (time.perf_counter() - t0) / steps
        byt = sum(layer_bytes(q.rows, q.cols, cfg, n) for q in ref_api_layers)
        out["e2e_reference_api"] = {
            "value": round(byt / dt / 1e9, 3), "unit": "GB/s", "ms_per_step": round(dt * 1e3, 3),
            "h2d_bytes_per_step": sum(2 * q.cols * n for q in ref_api_layers),
            "d2h_bytes_per_step": sum(4 * q.rows * n for q in ref_api_layers),
            "path": "per step: the 7 layers of one block, each codegemm_gemm(q, Matrix(x)) -> "
                    "(numpy y, OpCounters): host x copied in, one deterministic fused launch, "
                    "y copied out, synchronised; wall clock"}
    except Exception as e:
        out["e2e_reference_api"] = {"error": repr(e)[:200]}
    return out


# --------------------------------------------------------------------------- GPU
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", choices=("b200", "reference"), default="b200")
    ap.add_argument("--workload", choices=("auto", "8b", "70b"), default="auto")
    ap.add_argument("--config", choices=tuple(CONFIGS), default="m1v4g128")
    ap.add_argument("--batch", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--detail", action="store_true", help="also time every unique shape alone")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the config-1 / GQA / batch-sweep / reference-API lines")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test-only: the N > 1 code path with every rank on GPU 0 and gloo plumbing
    # (the fused exchange still runs between the processes over CUDA IPC; the
    # contexts time-slice, so timings are meaningless; NCCL-only lines skipped)
    one_gpu = os.environ.get("CG_BENCH_ONE_GPU") == "1" and world > 1
    if one_gpu:
        local_rank = 0
    if args.workload == "auto":
        args.workload = "8b" if world == 1 else "70b"
    cfg = CONFIGS[args.config]
    n = args.batch
    global TILING_U
    if TILING_U == 0:
        TILING_U = 4 // cfg["m"]  # measured: u=4 41.5 us/block vs u=2 43.6 vs u=1 57.4 (m1v4)
    spec = block_spec(args.workload)
    if args.warmup < 3:
        args.warmup = 3

    import torch
    import torch.distributed as dist

    if world > 1:
        torch.cuda.set_device(local_rank)
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    if args.impl == "reference":
        run_reference(args, spec, cfg, n, rank, world)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    import paper_2512_17970_b200 as cg
    from paper_2512_17970_b200.dist import (XCHG_PUSH, GatheredLayout, PeerExchange,
                                            ShardedLayer)
    from oracle import codegemm_oracle as orc

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    step_bytes = sum(layer_bytes(r, c, cfg, n) for (_, r, c) in spec)
    weight_bytes = sum(layer_bytes(r, c, cfg, n, with_io=False) for (_, r, c) in spec) // world
    copies = max(2, -(-3 * L2_BYTES // max(1, weight_bytes)))

    # ---- layers: `copies` distinct copies of the block, rows sharded over ranks.
    #      A block's inputs (the x of q,k,v) and its outputs are views of one
    #      contiguous buffer each, so the end-to-end step moves them with one copy
    #      each way.
    in_elems = sum(c * n for i, (_, r, c) in enumerate(spec) if STEP_XSRC[i] is None)
    blocks, xbufs, ybufs = [], [], []
    ref_api_layers = []  # copy 0's QuantizedLayers: the reference-API end-to-end leg
    for cp in range(copies):
        layers = []
        xbuf = torch.empty(in_elems, dtype=torch.float16, device=dev)
        ybuf = torch.empty(sum(-(-r // world) * world * n for (_, r, c) in spec),
                           dtype=torch.float32, device=dev)
        xo = yo = 0
        for idx, (name, rows, cols) in enumerate(spec):
            q = make_layer(rows, cols, cfg, layer_seed(cp, idx, rows, cols))
            if cp == 0 and world == 1:
                ref_api_layers.append(q)
            sl = (ShardedLayer(q, rank, world, u=TILING_U) if world > 1
                  else cg.DeviceLayer(q, u=TILING_U))
            x = torch.from_numpy(orc.bench_input_array(cols, n, cp * 31 + idx)).to(dev)
            if STEP_XSRC[idx] is None:
                xbuf[xo: xo + cols * n].copy_(x.view(-1))
                x = xbuf[xo: xo + cols * n].view(cols, n)
                xo += cols * n
            per = sl.per if world > 1 else rows
            y = ybuf[yo: yo + per * world * n].view(per * world, n)
            yo += per * world * n
            layers.append({"name": name, "rows": rows, "cols": cols, "layer": sl, "x": x,
                           "y_local": torch.empty((per, n), dtype=torch.float32, device=dev),
                           "y": y})
        blocks.append(layers)
        xbufs.append(xbuf)
        ybufs.append(ybuf)

    def dev_layer(L):
        return L["layer"].device_layer if world > 1 else L["layer"]

    # N > 1: the all-gather fused into the staged launch (cg_gemm_stages_xchg):
    # every layer's gathered output lives in one peer-mapped region per rank;
    # each stage's rows are stored into every peer's copy over NVLink and the
    # next stage reads the gathered x once every rank arrived
    if world > 1:
        glay = GatheredLayout([r for _ in blocks for (_, r, c) in spec], n, world)
        comm = PeerExchange(world, rank, glay.nbytes, timeout_ms=60000, device=local_rank)
        comm.connect()
        nl = len(spec)
        for cp, b in enumerate(blocks):
            for i, L in enumerate(b):
                L["g_local"] = glay.local(comm, cp * nl + i)
                L["g_full"] = glay.gathered(comm, cp * nl + i)
                assert L["g_local"].shape[0] == L["layer"].r1 - L["layer"].r0

    prepared = {}  # one prepared launch (marshalled once) per block copy

    def run_xchg(b):
        """The whole row-sharded block in ONE launch per rank, all-gathers fused in."""
        key = ("x", id(b))
        if key not in prepared:
            xs = [b[i]["x"] if src is None else b[src]["g_full"] for i, src in enumerate(STEP_XSRC)]
            prepared[key] = cg.StagedLaunch([dev_layer(L) for L in b], xs,
                                            [L["g_local"] for L in b], list(STEP_STAGES),
                                            xchg=[XCHG_PUSH] * len(b), comm=comm)
        prepared[key]()

    def run_kernel(L):
        dl = dev_layer(L)
        if dl is not None:
            dl.gemm(L["x"], L["y_local"] if world > 1 else L["y"])

    def run_layer(L):
        run_kernel(L)
        if world > 1:
            dist.all_gather_into_tensor(L["y"], L["y_local"])

    stream = torch.cuda.Stream(dev)

    def capture(fn):
        # warm the path (kernel attributes, NCCL communicators) outside capture
        with torch.cuda.stream(stream):
            fn()
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            fn()
        return g

    # A decode step launches what a decoder block can: layers that read the
    # same x go in one grouped launch ({q,k,v}, {o}, {gate,up}, {down}).
    groups = STEP_GROUPS

    def run_group(b, grp):
        dls = [dev_layer(b[i]) for i in grp]
        if all(d is not None for d in dls):
            cg.gemm_group(dls, [b[i]["x"] for i in grp],
                          [b[i]["y_local"] if world > 1 else b[i]["y"] for i in grp])
        if world > 1:
            for i in grp:
                dist.all_gather_into_tensor(b[i]["y"], b[i]["y_local"])

    def run_staged(b):
        """The whole block in one launch: stage chain with real data dependencies."""
        key = ("s", id(b))
        if key not in prepared:
            xs = [b[i]["x"] if src is None else b[src]["y"] for i, src in enumerate(STEP_XSRC)]
            prepared[key] = cg.StagedLaunch([L["layer"] for L in b], xs, [L["y"] for L in b],
                                            list(STEP_STAGES))
        prepared[key]()

    CHAIN = int(os.environ.get("CG_BENCH_CHAIN", "2"))  # blocks per launch (<= 16 layers)

    def run_staged_chain(j0):
        """CHAIN block copies, chained, in ONE persistent launch: block j's q,k,v read
        block j-1's y_down (a model's layer stack), stages 4j .. 4j+3."""
        lay, xs, ys, st = [], [], [], []
        for jj in range(CHAIN):
            j = (j0 + jj) % len(blocks)
            b = blocks[j]
            for i, src in enumerate(STEP_XSRC):
                lay.append(b[i]["layer"])
                if src is not None:
                    xs.append(b[src]["y"])
                else:
                    xs.append(b[i]["x"] if jj == 0 else blocks[(j - 1) % len(blocks)][len(spec) - 1]["y"])
                ys.append(b[i]["y"])
                st.append(len(groups) * jj + STEP_STAGES[i])
        cg.gemm_stages(lay, xs, ys, st)

    if world == 1:
        # one launch runs a step for every block copy (len(blocks) decoder
        # blocks chained: launch and grid-completion latency are paid once per
        # copy cycle); single-step launches make up a step count that is not
        # a multiple of the copy count
        nlaunch = len(blocks) // CHAIN
        graphs = [capture(lambda: [run_staged_chain(CHAIN * k) for k in range(nlaunch)])]
        # a step count that is not a multiple of the graph's: chained launches of
        # CHAIN copies first (the copies after the graph's, rotating on), then
        # single-block launches for what remains
        pairs = [capture(lambda j0=j0: run_staged_chain(j0))
                 for j0 in range(CHAIN * nlaunch, CHAIN * nlaunch + len(blocks), CHAIN)]
        singles = [capture(lambda b=b: run_staged(b)) for b in blocks]
        launches_per_step = 1.0 / CHAIN
    else:
        graphs = [capture(lambda b=b: run_xchg(b)) for b in blocks]
        singles = pairs = None
        launches_per_step = 1

    def timed(replays, count, per_graph=1):
        """Replay graphs[i % len] until `count` steps (per_graph steps per replay) ran;
        device ms (max over ranks)."""
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            # a ~0.1 ms spin kernel ahead of the start event (outside the timed
            # region): the host has queued the timed graphs by the time the start
            # event fires, so a short region does not time the host's first submit
            torch.cuda._sleep(200_000)
            ev0.record(stream)
            for i in range(count // per_graph):
                replays[i % len(replays)].replay()
            rem = count % per_graph  # exactly `count` steps
            for i in range(rem // CHAIN):
                pairs[i % len(pairs)].replay()
            for i in range(rem % CHAIN):
                singles[i].replay()
            ev1.record(stream)
        torch.cuda.synchronize(dev)
        ms = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
            dist.barrier()
        return ms

    # ---- warmup + timed region (clocks sampled during it)
    spg = (len(blocks) // CHAIN) * CHAIN if world == 1 else 1  # steps per graph replay
    timed(graphs, args.warmup, spg)
    soak = 0
    with ClockSampler(local_rank) as clk:
        ms = timed(graphs, args.steps, spg)
        if ms < 1000.0:  # too short for 50 ms sampling: keep the same load running ~1 s
            soak = int(args.steps * (1000.0 - ms) / max(ms, 1e-3)) + 1
            timed(graphs, soak, spg)
    clocks = clk.summary()
    if clocks is not None and soak:
        clocks["note"] = (f"timed region {ms:.1f} ms; sampling continued over {soak} more "
                          "identical steps right after it")
    ms_per_step = ms / args.steps
    value = step_bytes * args.steps / (ms / 1e3) / 1e9

    # ---- the same step with one launch per layer, and one launch per group
    reps = max(20, min(400, args.steps // 4))
    reps = -(-reps // spg) * spg
    ms_sep = ms_grp = None
    if not one_gpu:
        # (N=1: one graph over every block copy -- `nb` steps per replay)
        nb = len(blocks) if world == 1 else 1
        reps_nb = -(-reps // nb) * nb
        sep = [capture(lambda: [run_layer(L) for b in blocks for L in b])] if world == 1 else \
            [capture(lambda b=b: [run_layer(L) for L in b]) for b in blocks]
        timed(sep, 3 * nb, nb)
        ms_sep = timed(sep, reps_nb, nb) / reps_nb
        del sep
        if world == 1:
            grp = [capture(lambda: [run_group(b, g) for b in blocks for g in groups])]
        else:  # grouped launches + an NCCL all-gather per layer (the unfused path)
            grp = [capture(lambda b=b: [run_group(b, g) for g in groups]) for b in blocks]
        timed(grp, 3 * nb, nb)
        ms_grp = timed(grp, reps_nb, nb) / reps_nb
        del grp

    # ---- per-shape kernel microseconds: graphs of R back-to-back launches of
    #      one shape (rotating weight copies), so host launch cost is amortised
    uniq = []
    for idx, (name, rows, cols) in enumerate(spec):
        if name not in [u[0] for u in uniq]:
            uniq.append((name, idx, rows, cols))
    R = 4 * len(blocks)
    kern = {}
    for name, idx, rows, cols in uniq:
        if dev_layer(blocks[0][idx]) is None:
            continue
        gk = capture(lambda idx=idx: [run_kernel(blocks[r % len(blocks)][idx]) for r in range(R)])
        timed([gk], 2)
        kern[name] = (timed([gk], max(5, reps // R)) / (max(5, reps // R) * R) * 1e3, rows, cols,
                      idx)
        del gk
    us_per_layer = {f"{k} {v[1] // world}x{v[2]}": round(v[0], 3) for k, v in kern.items()}
    # staged chains: CH layers of one shape in ONE launch with a grid barrier
    # between consecutive layers (a dependent chain, as in a decode step);
    # chain k uses the shape's layer from block copies k, k+1, ... (distinct weights)
    us_chain = {}
    if world == 1:
        CH = min(7, len(blocks))
        for name, idx, rows, cols in uniq:
            def run_chain(k, idx=idx):
                c = [blocks[(k + r) % len(blocks)][idx] for r in range(CH)]
                cg.gemm_stages([L["layer"] for L in c], [L["x"] for L in c], [L["y"] for L in c],
                               list(range(CH)))

            gch = [capture(lambda: [run_chain(k) for k in range(len(blocks))])]
            nb = len(blocks)
            timed(gch, 2 * nb, nb)
            rr = max(2, reps // (CH * nb)) * nb
            us_chain[f"{name} {rows}x{cols}"] = round(timed(gch, rr, nb) / (rr * CH) * 1e3, 3)
            del gch
    # dominant kernel: the largest per-launch byte count (mlp_gate_up)
    dom = max(kern, key=lambda k: layer_bytes(kern[k][1] // world, kern[k][2], cfg, n))
    dom_us, dom_rows, dom_cols, dom_idx = kern[dom]
    dom_bytes = layer_bytes(-(-dom_rows // world), dom_cols, cfg, n)
    peaks_path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(peaks_path):
        peak, peak_src = float(json.load(open(peaks_path))["hbm_gbs"]), "measured"
    else:
        peak, peak_src = 6650.0, "fallback"
    achieved = dom_bytes / (dom_us * 1e-6) / 1e9
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(f"{args.config}:{dom_rows}x{dom_cols}")
        except Exception:
            traffic = None
    dl_dom = dev_layer(blocks[0][dom_idx])
    if world == 1:
        # one kernel per step: the staged block launch itself
        achieved = step_bytes / (ms_per_step * 1e-3) / 1e9
        traffic = None
        if os.path.exists(tpath):
            try:
                traffic = json.load(open(tpath)).get(f"{args.config}:block{args.workload}")
            except Exception:
                traffic = None
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": traffic,
                    "peak_source": peak_src,
                    "kernel": f"group_gemv_kernel<v{cfg['v']},m{cfg['m']},u{TILING_U}> staged "
                              f"launch, {CHAIN} chained blocks ({CHAIN * len(spec)} "
                              f"layers, {CHAIN * len(groups)} stages); per-step share",
                    "us_per_launch": round(ms_per_step * 1e3, 3),
                    "bytes_per_launch": step_bytes,
                    "frac_of_8TBs_nominal": round(achieved / 8000.0, 4),
                    "largest_layer_alone": {"layer": f"{dom} {dom_rows}x{dom_cols}",
                                            "us_per_launch": round(dom_us, 3),
                                            "GB/s": round(dom_bytes / (dom_us * 1e-6) / 1e9, 1)}}
    else:
        # one kernel per step per rank: the staged exchange launch over this
        # rank's rows (algorithmic bytes of its shards; x and gathered y included)
        rank_bytes = sum(layer_bytes(L["layer"].r1 - L["layer"].r0, L["cols"], cfg, n)
                         for L in blocks[0])
        achieved = rank_bytes / (ms_per_step * 1e-3) / 1e9
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "traffic": None,
                    "peak_source": peak_src,
                    "kernel": f"group_gemv_kernel<v{cfg['v']},m{cfg['m']},u{TILING_U}> staged "
                              f"exchange launch per rank ({len(spec)} row-sharded layers, "
                              f"{len(groups)} stages, all-gathers fused); per-GPU",
                    "us_per_launch": round(ms_per_step * 1e3, 3), "bytes_per_launch": rank_bytes,
                    "frac_of_8TBs_nominal": round(achieved / 8000.0, 4),
                    "largest_layer_alone": {"layer": f"{dom} {dom_rows // world}x{dom_cols}",
                                            "us_per_launch": round(dom_us, 3),
                                            "GB/s": round(dom_bytes / (dom_us * 1e-6) / 1e9, 1)}}

    # ---- end to end through the public API with host buffers
    e2e_steps = max(3, min(args.steps, 100))
    # one step = H2D of the step's inputs (x of q,k,v: one contiguous buffer) from
    # pinned memory, the staged launch (prepared), D2H of every layer's (gathered)
    # output (one contiguous range), synchronise
    host_x = torch.from_numpy(np.concatenate(
        [orc.bench_input_array(c, n, 100 + i).reshape(-1) for i, (_, r, c) in enumerate(spec)
         if STEP_XSRC[i] is None])).pin_memory()
    if world == 1:
        out_views = [ybufs[cp] for cp in range(len(blocks))]
    else:  # this block's gathered outputs: one range of the comm region
        nl = len(spec)
        out_views = []
        for cp in range(len(blocks)):
            a, z = glay.offset[cp * nl], glay.offset[cp * nl + nl - 1] + spec[-1][1] * n * 4
            out_views.append(comm.view(a, (z - a) // 4, 1).view(-1))
    host_y = torch.empty(out_views[0].numel(), dtype=torch.float32).pin_memory()
    h2d = host_x.numel() * 2
    d2h = host_y.numel() * 4

    for cp in range(len(blocks)):  # (plans are prepared outside the timed loop)
        run_staged(blocks[cp]) if world == 1 else run_xchg(blocks[cp])
    torch.cuda.synchronize(dev)
    e2e_stream = torch.cuda.current_stream(dev)
    if world == 1:
        # the kernel writes every layer's output straight into pinned host memory
        # once its stage completes (cg_stages_set_mirror): no D2H copy on the step's
        # critical path, the copies overlap the later stages
        def host_views(b):
            vs, off = [], 0
            for L in b:
                nel = L["y"].numel()
                vs.append(host_y[off: off + nel].view(L["y"].shape))
                off += nel
            return vs
        bound = [prepared[("s", id(blocks[cp]))].bind_host_mirrored(
            host_x, xbufs[cp], host_views(blocks[cp]), stream=e2e_stream)
            for cp in range(len(blocks))]
    else:
        bound = [prepared[("x", id(blocks[cp]))].bind_host(
            host_x, xbufs[cp], out_views[cp], host_y, stream=e2e_stream) for cp in range(len(blocks))]

    def e2e_step(cp):
        bound[cp]()

    for cp in range(len(blocks)):  # first calls build each copy's host graph, untimed
        e2e_step(cp)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for i in range(e2e_steps):
        e2e_step(i % len(blocks))
    torch.cuda.synchronize(dev)
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e = {"value": round(step_bytes * e2e_steps / e2e_s / 1e9, 3), "unit": "GB/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "ms_per_step": round(e2e_s / e2e_steps * 1e3, 3),
           "path": "per step: StagedLaunch.bind_host_mirrored(...)() (cg_stages_run_host with "
                   "cg_stages_set_mirror): one pinned H2D of the step inputs (q,k,v x), the prepared "
                   "staged launch, whose CTAs write all 7 layer outputs into pinned host memory as "
                   "each stage completes, sync; wall clock"
           if world == 1 else "per step: StagedLaunch.bind_host(...)(): one pinned H2D of the step "
                              "inputs, the prepared staged exchange launch, one pinned D2H of all "
                              "7 gathered outputs, sync; wall clock, max over ranks"}

    extras = {}
    if world == 1 and not args.no_extras:
        extras = measure_extras(args, cfg, n, blocks, spec, kern, ref_api_layers, peak, capture,
                                timed, stream, dev)

    base = base_c = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base, base_c = cpu_baseline(spec, cfg, n)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
            "vs_baseline": None, "dtype": "u8 codes, f16 in, f32 accumulate",
            "data": "synthetic (reference generators random_layer/bench_input; random codebooks, "
                    "codes, scales)",
            "config": bench_config(args, n, world),
            "setup": {"weight_copies": copies,
                      "l2": f"inputs larger than L2: {copies} distinct block copies rotated "
                            f"({copies * weight_bytes / 2**20:.0f} MiB of weights per rank)",
                      "parallelism": f"rows sharded over {world} GPUs, all-gathers fused "
                                     "into the kernel over NVLink peer stores"
                      if world > 1 else "single GPU",
                      "launch": ("one persistent staged launch (cg_gemm_stages) per "
                                 f"{CHAIN} steps: {CHAIN} block copies chained "
                                 "as a layer stack, each block the stages {q,k,v} -> {o} -> "
                                 "{gate,up} -> {down}; o/gate/up/down read the previous stage's "
                                 "y and the next block's q,k,v read y_down, rounded to fp16; "
                                 f"grid barriers between stages, u={TILING_U}; CUDA graph")
                      if world == 1 else
                      "per step: ONE staged exchange launch per rank (cg_gemm_stages_xchg): "
                      "stages {q,k,v} -> {o} -> {gate,up} -> {down}, every layer's rows "
                      "pushed to every peer after its stage, the next stage reading the "
                      "gathered y; CUDA graph per block copy, PDL"},
            "us_per_layer": us_per_layer,
            "us_per_layer_staged_chain": us_chain,
            "us_per_block": round(ms_per_step * 1e3, 3),
            "step_launches": [["stage %d: " % s + ",".join(spec[i][0] for i in g)
                               for s, g in enumerate(groups)]],
            "separate_launches": None if ms_sep is None else
            {"us_per_block": round(ms_sep * 1e3, 3),
                                  "value": round(step_bytes / (ms_sep / 1e3) / 1e9, 2),
                                  "launches_per_step": len(spec)},
            "grouped_launches": None if ms_grp is None else
            {"us_per_block": round(ms_grp * 1e3, 3),
                                 "value": round(step_bytes / (ms_grp / 1e3) / 1e9, 2),
                                 "launches_per_step": len(groups),
                                 "all_gather": None if world == 1 else "NCCL, one per layer"},
            "roofline": roofline,
            **extras,
            "cpu_baseline": base, "cpu_baseline_c": base_c,
            "e2e": e2e,
            "gpu_launches": (args.steps // spg * (spg // CHAIN) + (args.steps % spg) // CHAIN
                             + (args.steps % spg) % CHAIN) if world == 1
            else launches_per_step * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
