# instruction-cache behaviour of the C3 training kernel (one launch, 32 images)
M=sm__icc_requests.sum,sm__icc_requests_lookup_hit.sum,sm__icc_requests_lookup_miss_tag_miss.sum,sm__icc_requests_lookup_miss_tag_hit.sum,gcc__cache_requests_type_instruction.sum,gcc__average_cache_request_type_instruction_hit_rate.pct,lts__t_requests_srcunit_gcc.sum,gpu__time_duration.sum,sm__inst_executed.sum,smsp__pcsamp_warps_issue_stalled_no_instructions.sum,smsp__pcsamp_sample_count.sum
ncu --metrics $M --clock-control none -k regex:net_spec_kernel -c 1 -s 1 --csv python tools/ncu_one.py C3 32 > gpurun_out/icache_C3.csv 2>&1
CKB200_NO_SPEC=1 ncu --metrics $M --clock-control none -k regex:net_team_kernel -c 1 -s 1 --csv python tools/ncu_one.py C3 32 > gpurun_out/icache_C3_generic.csv 2>&1
CKB200_NO_SPEC=1 python bench.py --config C3 --blocks '' --no-cpu-baseline --no-e2e --no-committee --no-deform --no-tc --tc-train '' --steps 20 --warmup 5 2>/dev/null | tail -1 > gpurun_out/generic_C3.json
