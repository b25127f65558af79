#!/bin/bash
# One GPU measurement pass: bench line, launch list, full ncu capture of the
# persistent training kernel.  Usage (under gpurun): bash tools/gpu_round.sh TAG [CONFIG]
set -u
TAG=${1:-r01}
CFG=${2:-C2}
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python bench.py --config $CFG > $OUT/bench_${TAG}_${CFG}.json 2> $OUT/bench_${TAG}_${CFG}.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_${TAG}_${CFG}.csv \
  python bench.py --config $CFG --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-committee > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"net_(team|spec)" -s 1 -c 1 \
  -o $OUT/prof_${TAG}_${CFG} -f \
  python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-committee > $OUT/ncu_${TAG}_${CFG}.log 2>&1
echo done
