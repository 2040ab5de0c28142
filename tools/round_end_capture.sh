#!/bin/bash
# Bench + reference arm + ncu evidence for profiles/ (run on the GPU box from the repo root).
set -u
mkdir -p gpurun_out
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
# launch list of the timed encode kernels (cold-cache, serialised: shares only)
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"beam_fast|table_tc|sgemm_table|bound_prep|cb_tf32_prep" -c 60 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-anneal --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "launch rc=$?"
# full captures: the dominant kernel (L=10 gather filter), the tcgen05 score table, the assign pair
ncu --set full --clock-control none --import-source on -k regex:beam_fast -c 1 -o gpurun_out/prof_beam_fast -f \
    python tools/prof_tc.py 2 10 > gpurun_out/ncu_bf.log 2>&1; echo "full bf rc=$?"
ncu --set full --clock-control none --import-source on -k regex:table_tc -c 1 -o gpurun_out/prof_table_tc -f \
    python tools/prof_tc.py 2 10 > gpurun_out/ncu_tt.log 2>&1; echo "full table rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"assign_tc_kernel|assign_recheck|x_tf32_prep" -c 3 -o gpurun_out/prof_assign -f \
    python tools/bench_assign.py 1000000 128 > gpurun_out/ncu_as.log 2>&1; echo "full assign rc=$?"
ncu -i gpurun_out/prof_beam_fast.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/bf_source.csv 2>/dev/null
