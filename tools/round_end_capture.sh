#!/bin/bash
# Bench + reference arm + ncu evidence for profiles/ (run on the GPU box from the repo root).
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
# launch list of the timed encode kernels (cold-cache, serialised: shares only)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"beam_fast|table_tc|a_tf32_img|sgemm_table|bound_prep|cb_tf32_prep|greedy|beam_pair" -c 60 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-anneal --no-cpu --no-adc --no-atree > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
# full captures: L=10 beam kernel, tcgen05 score table, L=1 greedy kernel, ADC scan
timeout 600 ncu --set full --clock-control none --import-source on -k regex:beam_fast -c 1 -o gpurun_out/prof_beam_fast -f \
    python tools/prof_tc.py 2 10 > gpurun_out/ncu_bf.log 2>&1; echo "full bf rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"table_tc_stream|a_tf32_img|greedy" -c 4 -o gpurun_out/prof_l1 -f \
    python tools/prof_tc.py 2 1 > gpurun_out/ncu_l1.log 2>&1; echo "full l1 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adc_scan_packed -c 1 -o gpurun_out/prof_adc -f \
    python tools/bench_adc.py 100000000 2000 100000 > gpurun_out/ncu_adc.log 2>&1; echo "full adc rc=$?"
# config C (D=960): D-tiled tcgen05 table + wide-row greedy kernel
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"greedy|table_tc_stream|a_tf32_img" -c 3 -o gpurun_out/prof_c -f \
    python tools/prof_configc.py 1 > gpurun_out/ncu_c.log 2>&1; echo "full configC rc=$?"
for r in prof_beam_fast prof_l1 prof_adc prof_c; do
  ncu -i gpurun_out/$r.ncu-rep --page raw --csv > gpurun_out/${r}_raw.csv 2>/dev/null
done
ncu -i gpurun_out/prof_beam_fast.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/bf_source.csv 2>/dev/null
ncu -i gpurun_out/prof_l1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/l1_source.csv 2>/dev/null
rm -f gpurun_out/*.ncu-rep
