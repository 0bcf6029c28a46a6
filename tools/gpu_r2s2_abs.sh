# A/B timing at small L (K steps per launch is what bench uses; step_time is one launch per step)
mkdir -p gpurun_out
v=$1
for L in 16383 65535 1048575; do
  st=20; [ $L = 1048575 ] && st=10
  timeout 600 python tools/ab_time.py build_ablate/lib_base.so build_ablate/lib_$v.so 3 -- --length $L --walks 444 --steps $st --mode auto
done > gpurun_out/abs_$v.txt 2>&1
cat gpurun_out/abs_$v.txt
timeout 900 python -m pytest tests -q -m gpu -x -k "cert or phase2 or smoke or parity" > gpurun_out/abs_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/abs_pytest.log
