python tools/subprof.py C3 0,100 > gpurun_out/sub_C3_scatter.txt 2>&1
CKB200_PULL=gather python tools/subprof.py C3 0,100,147 > gpurun_out/sub_C3_gather.txt 2>&1
CKB200_PULL=gather python tools/phases.py C3 > gpurun_out/ph_C3_gather.txt 2>&1
python tools/phases.py C3 > gpurun_out/ph_C3_scatter.txt 2>&1
