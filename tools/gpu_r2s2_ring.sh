mkdir -p gpurun_out
for v in r3 r4; do
for L in 1048575 65535; do
  st=20; [ $L = 1048575 ] && st=10
  timeout 600 python tools/ab_time.py build_ablate/lib_base.so build_ablate/lib_$v.so 3 -- --length $L --walks 444 --steps $st --mode auto
done
done > gpurun_out/ring.txt 2>&1
cat gpurun_out/ring.txt
PSLB200_LIB=build_ablate/lib_r4.so timeout 900 python -m pytest tests -q -m gpu -x -k "cert or phase2 or smoke" > gpurun_out/ring_pytest.log 2>&1; echo pytest_r4=$?; tail -1 gpurun_out/ring_pytest.log
