# ncu --set full capture of the gather-filter beam kernel (65,536 config-B vectors, L=10)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:beam_fast -c 1 -o gpurun_out/prof_bf -f python tools/prof_tc.py 2 10 > gpurun_out/ncu_bf.log 2>&1; echo "bf rc=$?"
ncu -i gpurun_out/prof_bf.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/bf_source.csv 2>/dev/null
ncu -i gpurun_out/prof_bf.ncu-rep --page raw --csv > gpurun_out/bf_raw.csv 2>/dev/null
