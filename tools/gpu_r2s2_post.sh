# after the long run: epilogue change A/B (base = HEAD, ep = working tree) + parity, then issuer-warp ablations
mkdir -p gpurun_out
for L in 16383 65535 1048575; do
  st=20; [ $L = 1048575 ] && st=10
  timeout 600 python tools/ab_time.py build_ablate/lib_base.so build_ablate/lib_ep.so 3 -- --length $L --walks 444 --steps $st --mode auto
done > gpurun_out/post_ep.txt 2>&1
cat gpurun_out/post_ep.txt
PSLB200_LIB=build_ablate/lib_ep.so timeout 900 python -m pytest tests -q -m gpu -x -k "cert or phase2 or smoke or parity" > gpurun_out/post_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/post_pytest.log
for v in fac nox15 nox14 nox12; do
  timeout 600 python tools/ab_time.py build_ablate/lib_ep.so build_ablate/lib_$v.so 2 > gpurun_out/post_$v.txt 2>&1; tail -1 gpurun_out/post_$v.txt
done
