mkdir -p gpurun_out
for v in t6 t10; do
  timeout 600 python tools/ab_time.py build_ablate/lib_base.so build_ablate/lib_$v.so 3 -- --length 1048575 --walks 444 --steps 10 --mode auto
done > gpurun_out/tail.txt 2>&1
cat gpurun_out/tail.txt
