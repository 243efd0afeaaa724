timeout 900 python tools/sweep.py batch > gpurun_out/sweep_batch.jsonl 2> gpurun_out/sweep_batch.err; tail -2 gpurun_out/sweep_batch.err
timeout 900 python tools/sweep.py hyper > gpurun_out/sweep_hyper.jsonl 2> gpurun_out/sweep_hyper.err; tail -2 gpurun_out/sweep_hyper.err
cat gpurun_out/sweep_batch.jsonl gpurun_out/sweep_hyper.jsonl
