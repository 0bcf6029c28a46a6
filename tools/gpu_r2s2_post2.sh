mkdir -p gpurun_out
for v in vall vnou; do
for L in 1048575 16383; do
  st=20; [ $L = 1048575 ] && st=10
  timeout 600 python tools/ab_time.py build_ablate/lib_base.so build_ablate/lib_$v.so 3 -- --length $L --walks 444 --steps $st --mode auto
done
done > gpurun_out/post2.txt 2>&1
cat gpurun_out/post2.txt
