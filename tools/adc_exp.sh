mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q -k "adc or atree" 2>&1 | tail -2
for U in 4 8 2; do
  if [ $U != 4 ]; then touch paper_1509_05194_b200/csrc/ops.cu; make -C paper_1509_05194_b200/csrc EXTRA=-DDA_ADC_U=$U > /dev/null 2>&1; fi
  echo "U=$U"; timeout 300 python tools/bench_adc.py 1e9 10000 100000 2>&1 | grep packed
done
