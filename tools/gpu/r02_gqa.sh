for e in "" "CG_DEBUG_FLAGS=524288" "" "CG_DEBUG_FLAGS=524288"; do
  env $e timeout 900 python bench.py --no-cpu-baseline --steps 300 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('[$e]', d['us_per_block'], 'gqa', d['gqa_block']['us_per_block'], 'indep', d['independent_layers']['us_per_block'], 'cfg1', d['config1_layer']['us_per_launch'], 'b4', d['batch_sweep'][0]['us_per_block'])"
done
