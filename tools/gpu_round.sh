#!/bin/bash
# One GPU measurement pass (run under gpurun): bench lines for C1-C4, the ncu
# launch list of the C2 bench, and --set full captures of the persistent
# training kernel (C2), a tensor-core eval GEMM (C4 conv2) and the deformation
# kernel.  Usage: bash tools/gpu_round.sh TAG
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python bench.py --config C2 > $OUT/bench_${TAG}_C2.json 2> $OUT/bench_${TAG}_C2.err
for c in C1 C3 C4; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > $OUT/bench_${TAG}_$c.json 2> $OUT/bench_${TAG}_$c.err
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_${TAG}_C2.csv \
  python bench.py --config C2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-committee > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"net_(team|spec)" -s 1 -c 1 \
  -o $OUT/prof_${TAG}_C2 -f \
  python bench.py --config C2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-committee --no-deform > $OUT/ncu_${TAG}_C2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 1 -c 1 \
  -o $OUT/prof_${TAG}_tc_C4 -f python tools/tc_launches.py C4 3 > $OUT/ncu_${TAG}_tc.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:deform_kernel -c 1 \
  -o $OUT/prof_${TAG}_deform -f \
  python bench.py --config C1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --no-committee > $OUT/ncu_${TAG}_deform.log 2>&1
echo done
