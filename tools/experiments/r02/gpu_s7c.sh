mkdir -p gpurun_out/s7c
export NCU_DIR=gpurun_out/s7c
SKIP=3 timeout 900 bash tools/prof.sh fan 'apply_fan' --config 1 --graph off > gpurun_out/s7c/prof_fan.txt 2>&1; head -c 1500 gpurun_out/s7c/prof_fan.txt; echo
python tools/ncu_sass_hot.py gpurun_out/s7c/fan.ncu-rep 45 > gpurun_out/s7c/fan_hot.txt 2>&1; head -70 gpurun_out/s7c/fan_hot.txt
cp gpurun_out/fan_by_opcode.txt gpurun_out/s7c/
