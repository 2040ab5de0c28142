# ncu --set full capture of the assign recheck kernel (1M rows, d=128)
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:assign_recheck -c 1 -o gpurun_out/prof_rc -f python tools/bench_assign.py 1000000 128 > gpurun_out/ncu_rc.log 2>&1; echo "rc rc=$?"
ncu -i gpurun_out/prof_rc.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/rc_source.csv 2>/dev/null
ncu -i gpurun_out/prof_rc.ncu-rep --page raw --csv > gpurun_out/rc_raw.csv 2>/dev/null
