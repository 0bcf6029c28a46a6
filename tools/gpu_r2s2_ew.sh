mkdir -p gpurun_out
for L in 1048575 65535; do
  st=20; [ $L = 1048575 ] && st=10
  timeout 600 python tools/ab_time.py build_ablate/lib_base.so build_ablate/lib_ew.so 3 -- --length $L --walks 444 --steps $st --mode auto
done > gpurun_out/ew.txt 2>&1
cat gpurun_out/ew.txt
