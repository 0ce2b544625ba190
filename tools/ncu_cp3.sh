set -x
CMD="python bench.py --config 4 --iters 3"
timeout 1500 ncu --set full --clock-control none --import-source on \
  --metrics sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active \
  -k regex:"vest_cp_3" -s 1 -c 1 \
  -o gpurun_out/r2c_cp3 $CMD > gpurun_out/ncu_cp3.log 2>&1
tail -3 gpurun_out/ncu_cp3.log
ncu -i gpurun_out/r2c_cp3.ncu-rep --page raw --csv > gpurun_out/r2c_cp3_raw.csv
ncu -i gpurun_out/r2c_cp3.ncu-rep --page source --csv > gpurun_out/r2c_cp3_source.csv 2>/dev/null
ncu -i gpurun_out/r2c_cp3.ncu-rep --page details > gpurun_out/r2c_cp3_details.txt 2>/dev/null
ls -la gpurun_out/
if [ $(stat -c %s gpurun_out/r2c_cp3.ncu-rep) -gt 30000000 ]; then rm gpurun_out/r2c_cp3.ncu-rep; fi
