mkdir -p gpurun_out
for v in "$@"; do
  timeout 600 python tools/ab_time.py build_ablate/lib_base.so build_ablate/lib_$v.so ${ROUNDS:-2} > gpurun_out/ab_$v.txt 2>&1
  tail -2 gpurun_out/ab_$v.txt
done
