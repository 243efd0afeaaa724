# contiguous task ranges + Psumbook reuse: tests, A/B (CG_NO_CONTIG=1) on indep + chain
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/contig_tests.txt 2>&1; tail -3 gpurun_out/contig_tests.txt
for a in "8b 4" "70b 4"; do timeout 300 python tools/indep_block.py $a; CG_NO_CONTIG=1 timeout 300 python tools/indep_block.py $a; done > gpurun_out/contig_indep.jsonl 2> gpurun_out/contig_indep.err
cat gpurun_out/contig_indep.jsonl; tail -3 gpurun_out/contig_indep.err
for e in "" "CG_NO_CONTIG=1"; do env $e timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 500 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$e', d['us_per_block'], d['roofline']['frac'])"; done
for e in "" "CG_NO_CONTIG=1"; do env $e timeout 600 python bench.py --workload 70b --no-cpu-baseline --no-extras --steps 200 --warmup 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('70b $e', d['us_per_block'], d['roofline']['frac'])"; done
INDEP=1 timeout 120 python tools/stamps_block.py 1 > gpurun_out/stamps_indep1_contig.txt 2>&1; head -40 gpurun_out/stamps_indep1_contig.txt
