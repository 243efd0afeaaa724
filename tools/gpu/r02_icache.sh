# ncu full capture of the chained block (current library): per-SASS executed counts and stall samples
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:group_gemv -s 2 -c 1 -o gpurun_out/prof_ic -f python tools/profile_block.py 4 > /dev/null 2>&1
ncu -i gpurun_out/prof_ic.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_ic_sass.csv 2>/dev/null
ncu -i gpurun_out/prof_ic.ncu-rep --page raw --csv > gpurun_out/prof_ic_raw.csv 2>/dev/null
rm -f gpurun_out/prof_ic.ncu-rep
gzip -f gpurun_out/prof_ic_sass.csv
ls -la gpurun_out/prof_ic*
