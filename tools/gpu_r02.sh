#!/bin/bash
# Round-2 measurement pass (under gpurun): the GPU test suite, smoke, the
# default bench line + the reference arm, the ncu launch list of the headline
# bench, --set full captures (+ instruction-mix / L2 counters) of the C3 and C2
# training kernels, a tensor-core eval GEMM and a tensor-core training GEMM,
# summarised by tools/ncu_counters.py; phase budgets of C1-C4'.
# Usage: bash tools/gpu_r02.sh TAG
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_${TAG}.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_${TAG}.log 2>&1
timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench_${TAG}.json 2> $OUT/bench_${TAG}.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/ref_${TAG}.json 2> $OUT/ref_${TAG}.err
timeout 300 python tools/phases.py C1 C2 C3 C4 C4F > $OUT/phases_${TAG}.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches_${TAG}_C3.csv \
  python bench.py --steps 2 --warmup 1 --blocks "" --no-cpu-baseline --no-e2e --no-committee \
  --no-deform > /dev/null 2>&1
EXTRA=sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
for c in C3 C2; do
  timeout 600 ncu --set full --metrics $EXTRA --clock-control none --import-source on \
    -k regex:net_spec -s 1 -c 1 -o $OUT/prof_${TAG}_$c -f \
    python bench.py --config $c --steps 1 --warmup 1 --blocks "" --no-cpu-baseline --no-e2e \
    --no-committee --no-deform --no-tc > $OUT/ncu_${TAG}_$c.log 2>&1
  python tools/ncu_counters.py $OUT/prof_${TAG}_$c.ncu-rep --label "train $c 128 img" \
    > $OUT/counters_${TAG}_$c.json 2>> $OUT/ncu_${TAG}_$c.log
done
timeout 600 ncu --set full --metrics $EXTRA --clock-control none --import-source on \
  -k regex:gemm_kernel -s 1 -c 1 -o $OUT/prof_${TAG}_tc_C4 -f python tools/tc_launches.py C4 3 \
  > $OUT/ncu_${TAG}_tc.log 2>&1
python tools/ncu_counters.py $OUT/prof_${TAG}_tc_C4.ncu-rep --label "tc eval C4 conv2" \
  > $OUT/counters_${TAG}_tc_C4.json 2>> $OUT/ncu_${TAG}_tc.log
CKB200_TCT_NOGRAPH=1 timeout 600 ncu --set full --metrics $EXTRA --clock-control none \
  -k regex:tgemm -s 8 -c 2 -o $OUT/prof_${TAG}_tct_C4F -f python tools/tct_one.py C4F \
  > $OUT/ncu_${TAG}_tct.log 2>&1
python tools/ncu_counters.py $OUT/prof_${TAG}_tct_C4F.ncu-rep --label "tc training C4F" \
  > $OUT/counters_${TAG}_tct_C4F.json 2>> $OUT/ncu_${TAG}_tct.log
echo done
