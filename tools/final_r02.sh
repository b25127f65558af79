# final round-2 numbers with the committed build: bench line, reference arm, phase budgets,
# launch list of the headline bench, sub-phase timers of C3
set -u
OUT=gpurun_out; TAG=${1:-r02z}
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench_${TAG}.json 2> $OUT/bench_${TAG}.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/ref_${TAG}.json 2> $OUT/ref_${TAG}.err
timeout 300 python tools/phases.py C1 C2 C3 C4 C4F > $OUT/phases_${TAG}.txt 2>&1
timeout 300 python tools/subprof.py C3 0,100 > $OUT/sub_${TAG}_C3.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_${TAG}_C3.csv \
  python bench.py --steps 2 --warmup 1 --blocks "" --no-cpu-baseline --no-e2e --no-committee \
  --no-deform > /dev/null 2>&1
echo done
