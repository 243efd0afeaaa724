timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python - <<'PY'
import sys; sys.path.insert(0, ".")
import paper_2512_17970_b200 as cg
q = cg.random_layer(14336, 4096, cg.QuantConfig(v=4, m=1, b=6, g=128), seed=1)
dl = cg.DeviceLayer(q); print("m1v4b6 info", {k: dl.info[k] for k in ("fast_supported", "u", "device_bytes", "algorithmic_bytes")})
PY
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:group_gemv -s 3 -c 1 --csv python tools/profile_layer.py --rows 14336 --cols 4096 --config m1v4b6g128 --iters 5 2>/dev/null | grep -E "dram__bytes_read|gpu__time" | awk -F'","' '{print $(NF-2), $NF}'
timeout 600 python tools/sweep.py hyper 2>&1 | grep b6
