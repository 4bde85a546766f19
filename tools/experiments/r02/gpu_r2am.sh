# K2w at config 4 after the producer split: ncu
mkdir -p gpurun_out/r2am
NCU_DIR=gpurun_out/r2am timeout 1500 bash tools/prof.sh w4b apply_wide --config 4
