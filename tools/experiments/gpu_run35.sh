SKIP=3 timeout 600 bash tools/prof.sh fan1 'apply_fan' --config 1 --graph off > gpurun_out/prof_fan1.txt 2>&1; head -c 1500 gpurun_out/prof_fan1.txt; echo; head -16 gpurun_out/fan1_by_opcode.txt
