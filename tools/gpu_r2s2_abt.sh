# A/B timing (m20 and m16) + a parity subset on the default build
mkdir -p gpurun_out
for v in "$@"; do
  timeout 600 python tools/ab_time.py build_ablate/lib_base.so build_ablate/lib_$v.so ${ROUNDS:-3} > gpurun_out/ab_$v.txt 2>&1
  timeout 600 python tools/ab_time.py build_ablate/lib_base.so build_ablate/lib_$v.so 2 -- --length 65535 --walks 444 --steps 20 --mode auto >> gpurun_out/ab_$v.txt 2>&1
  cat gpurun_out/ab_$v.txt
done
timeout 900 python -m pytest tests -q -m gpu -x -k "cert or phase2 or smoke or parity" > gpurun_out/abt_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/abt_pytest.log
