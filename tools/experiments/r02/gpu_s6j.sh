mkdir -p gpurun_out/s6j
timeout 900 python tests/stress/repro_rowblocks.py 2000 150001 60 quant_lut=1 > gpurun_out/s6j/lut1.log 2>&1; tail -12 gpurun_out/s6j/lut1.log
timeout 900 python tests/stress/repro_rowblocks.py 2000 150001 60 quant_lut=0 > gpurun_out/s6j/lut0.log 2>&1; tail -6 gpurun_out/s6j/lut0.log
timeout 900 python tests/stress/repro_rowblocks.py 500 620001 30 quant_lut=1 > gpurun_out/s6j/f500.log 2>&1; tail -6 gpurun_out/s6j/f500.log
