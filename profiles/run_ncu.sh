#!/bin/bash
# ncu recipe (run under gpurun on one B200): the launch list of one bench step
# (cold-cache, serialised per-launch times) and a full capture of the top
# kernels.  Summaries are extracted by profiles/summarize_ncu.py into profiles/.
set -e
CMD="python bench.py --steps 1 --warmup 1 --no-cpu"
mkdir -p gpurun_out
$CMD > gpurun_out/plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launches.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on \
    --metrics sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active \
    -k regex:"${NCU_KERNELS:-k_rowpass|k_core_sall|k_sall_gemm|k_core_rpass|k_core_solve_g}" -s ${NCU_SKIP:-0} -c ${NCU_COUNT:-8} \
    -o gpurun_out/prof_full $CMD > gpurun_out/ncu_full.log 2>&1
