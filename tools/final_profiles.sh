#!/bin/bash
# Round-end measurement set on one B200 (run under gpurun): the headline bench
# line, the reference arm, every BASELINE config, the shard emulation of the
# headline config, the ncu launch list of the headline command and the full
# capture of config 4's steady-state kernels.  Everything lands in gpurun_out/.
set -x
python bench.py > gpurun_out/bench_default.log 2> gpurun_out/bench_default.err
tail -c 300 gpurun_out/bench_default.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.log 2> gpurun_out/bench_reference.err
rm -f gpurun_out/configs.jsonl gpurun_out/configs_graphs.jsonl gpurun_out/shard.jsonl
for c in 1 2 3 4 5; do python bench.py --config $c --iters 6 2>/dev/null | grep '^{' >> gpurun_out/configs.jsonl; done
for c in 1 2 3; do python bench.py --config $c --iters 12 --no-families 2>/dev/null | grep '^{' >> gpurun_out/configs_graphs.jsonl; done
for w in 2 4 8; do python bench.py --config 4 --iters 4 --shard-emulate $w 2>/dev/null | grep '^{' >> gpurun_out/shard.jsonl; done
python bench.py --steps 2 --warmup 3 --no-cpu --secondary 0 > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --secondary 0 > gpurun_out/ncu_launches.log 2>&1
bash tools/ncu_config4.sh
ls -la gpurun_out
