"""Cost of the fused row-shard exchange (cg_gemm_stages_xchg) on one GPU.

One decoder block (bench.py's staged chain {q,k,v} -> {o} -> {gate,up} ->
{down}, every layer's rows pushed) timed as:
  plain    : cg_gemm_stages, no exchange (bench.py's N=1 step)
  world1   : the same launch through a world-1 comm (counters, final barrier)
  worldW   : W in-process ranks on this GPU, each on sms/W CTAs with 1/W of
             every layer's rows, launched concurrently (one stream per rank,
             graph fork/join); every stage waits for every rank's pushed rows.
The W-rank line does the same total work as `plain` on the same SMs, so its
difference to `plain` is what the exchange (and the smaller grids) cost.
CUDA graphs over `copies` rotating block copies (> L2).

    python tools/xchg_bench.py [8b|70b] [m1v4g128]
"""

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import paper_2512_17970_b200 as cg  # noqa: E402
from paper_2512_17970_b200 import dist as cgd  # noqa: E402
from oracle import codegemm_oracle as orc  # noqa: E402


def main():
    workload = sys.argv[1] if len(sys.argv) > 1 else "8b"
    cfgname = sys.argv[2] if len(sys.argv) > 2 else "m1v4g128"
    cfg = bench.CONFIGS[cfgname]
    spec = bench.block_spec(workload)
    u = 4 // cfg["m"]
    n = 1
    dev = torch.device("cuda", 0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    step_bytes = sum(bench.layer_bytes(r, c, cfg, n) for (_, r, c) in spec)
    wbytes = sum(bench.layer_bytes(r, c, cfg, n, with_io=False) for (_, r, c) in spec)
    copies = max(2, -(-3 * bench.L2_BYTES // wbytes))
    qs = [[bench.make_layer(r, c, cfg, bench.layer_seed(cp, i, r, c))
           for i, (_, r, c) in enumerate(spec)] for cp in range(copies)]
    xs0 = [[torch.from_numpy(orc.bench_input_array(c, n, cp * 31 + i)).to(dev)
            for i, (_, r, c) in enumerate(spec)] for cp in range(copies)]
    stages = list(bench.STEP_STAGES)
    src = bench.STEP_XSRC
    out = {"workload": workload, "config": cfgname, "copies": copies}

    def time_graph(g, steps):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for _ in range(3):
                g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            e0.record(s)
            for _ in range(steps):
                g.replay()
            e1.record(s)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / (steps * copies) * 1e3  # us per block

    # plain staged launch
    layers = [[cg.DeviceLayer(q, u=u) for q in qb] for qb in qs]
    ys = [[torch.empty((r, n), dtype=torch.float32, device=dev) for (_, r, c) in spec]
          for _ in range(copies)]

    def plain(cp):
        x = [xs0[cp][i] if s_ is None else ys[cp][s_] for i, s_ in enumerate(src)]
        cg.gemm_stages(layers[cp], x, ys[cp], stages)

    def capture(fn):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            fn()
        return g

    g = capture(lambda: [plain(cp) for cp in range(copies)])
    out["plain_us"] = round(time_graph(g, 40), 2)
    del g

    for world in (1, 2, 4):
        lay = cgd.GatheredLayout([r for _ in range(copies) for (_, r, c) in spec], n, world)
        comms = [cgd.PeerExchange(world, r, lay.nbytes, ctas=sms // world if world > 1 else 0,
                                  timeout_ms=20000) for r in range(world)]
        cgd.PeerExchange.link(comms)
        nl = len(spec)
        rl = [[[cg.DeviceLayer(q, u=u, row_range=lay.bounds(cp * nl + i, r))
                for i, q in enumerate(qs[cp])] for cp in range(copies)] for r in range(world)]
        views = [[[(lay.local(comms[r], cp * nl + i), lay.gathered(comms[r], cp * nl + i))
                   for i in range(nl)] for cp in range(copies)] for r in range(world)]
        streams = [torch.cuda.Stream() for _ in range(world)]

        def step(cp):
            main = torch.cuda.current_stream()
            for r in range(world):
                streams[r].wait_stream(main)
                with torch.cuda.stream(streams[r]):
                    v = views[r][cp]
                    x = [xs0[cp][i] if s_ is None else v[s_][1] for i, s_ in enumerate(src)]
                    cg.gemm_stages(rl[r][cp], x, [a for a, _ in v], stages,
                                   xchg=[cgd.XCHG_PUSH] * nl, comm=comms[r])
            for r in range(world):
                main.wait_stream(streams[r])

        g = capture(lambda: [step(cp) for cp in range(copies)])
        us = time_graph(g, 40)
        out[f"world{world}_us"] = round(us, 2)
        # parity of the gathered outputs against the plain launch (tolerance: reduce-add mode)
        torch.cuda.synchronize()
        worst = 0.0
        for r in range(world):
            for i in range(nl):
                a = views[r][copies - 1][i][1].float()
                b = ys[copies - 1][i]
                worst = max(worst, float((a - b).norm() / b.norm()))
        out[f"world{world}_rel_l2_vs_plain"] = worst
        del g
        for c in comms:
            c.close()
    out["plain_GBps"] = round(step_bytes / (out["plain_us"] * 1e-6) / 1e9, 1)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
