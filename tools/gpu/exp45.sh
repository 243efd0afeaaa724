timeout 800 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/sweep.py batch > gpurun_out/sweep_batch.jsonl 2> gpurun_out/sweep_batch.err; tail -2 gpurun_out/sweep_batch.err
cut -c1-200 gpurun_out/sweep_batch.jsonl
