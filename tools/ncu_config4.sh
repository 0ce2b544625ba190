#!/bin/bash
# Full ncu capture of config 4's steady-state kernels (third iteration: the
# NVRTC kernels): vest_sd_1, k_rowpass_delta, k_core_hsample, vest_cp_3.
# Run under gpurun on one B200; writes the raw CSV page (and the report when
# it is small enough to travel) into gpurun_out/.
set -x
CMD="python bench.py --config 4 --iters 3"
$CMD > gpurun_out/c4_plain.log 2>&1 || exit 1
timeout 1500 ncu --set full --clock-control none \
  --metrics sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active \
  -k regex:"vest_sd_1|vest_cp_3|k_rowpass_delta|k_core_hsample" -s ${NCU_SKIP:-27} -c ${NCU_COUNT:-8} \
  -o gpurun_out/r2b_c4_full $CMD > gpurun_out/ncu_c4_full.log 2>&1
tail -3 gpurun_out/ncu_c4_full.log
ncu -i gpurun_out/r2b_c4_full.ncu-rep --page raw --csv > gpurun_out/r2b_c4_full_raw.csv
ls -la gpurun_out/
if [ $(stat -c %s gpurun_out/r2b_c4_full.ncu-rep) -gt 40000000 ]; then rm gpurun_out/r2b_c4_full.ncu-rep; fi
