mkdir -p gpurun_out
timeout 900 python tools/ab_time.py build_ablate/lib_base.so build_ablate/lib_$1.so 3 > gpurun_out/ab_$1.txt 2>&1; echo ab=$?
cat gpurun_out/ab_$1.txt
