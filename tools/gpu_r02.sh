#!/bin/bash
# Round-2 measurement pass (under gpurun): phase budgets, sub-phase timers,
# ncu counter captures of the training kernel (C3 headline, C2) with the
# instruction-mix / L2 metrics, summarised by tools/ncu_counters.py.
# Usage: bash tools/gpu_r02.sh TAG
set -u
TAG=${1:-r02}
OUT=gpurun_out
mkdir -p $OUT
EXTRA=sm__sass_thread_inst_executed_op_ffma_pred_on.sum,sm__sass_thread_inst_executed_op_fadd_pred_on.sum,sm__sass_thread_inst_executed_op_fmul_pred_on.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,lts__t_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 300 python tools/phases.py C1 C2 C3 C4 C4F > $OUT/phases_${TAG}.txt 2>&1
timeout 300 python tools/subprof.py C3 0,40,100 > $OUT/sub_${TAG}.txt 2>&1
for c in C3 C2; do
  timeout 600 ncu --set full --metrics $EXTRA --clock-control none --import-source on \
    -k regex:net_spec -s 1 -c 1 -o $OUT/prof_${TAG}_$c -f \
    python bench.py --config $c --steps 1 --warmup 1 --blocks "" --no-cpu-baseline --no-e2e \
    --no-committee --no-deform --no-tc > $OUT/ncu_${TAG}_$c.log 2>&1
  python tools/ncu_counters.py $OUT/prof_${TAG}_$c.ncu-rep --label "train $c 128 img" \
    > $OUT/counters_${TAG}_$c.json 2>> $OUT/ncu_${TAG}_$c.log
done
echo done
