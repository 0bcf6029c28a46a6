mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x -k "cert or phase2 or smoke or parity" > gpurun_out/b_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/b_pytest.log
timeout 600 python tools/small_l.py --length 16383 65535 262143 --walks 444 --steps 20 > gpurun_out/b_small.jsonl 2> gpurun_out/b_small.err; echo small=$?
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --exact-steps 0 > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; echo bench=$?
for L in 16383 1048575; do
  PSLB200_LIB=build_ablate/lib_pt.so timeout 300 python tools/pt_run.py 10 $L > gpurun_out/bpt_$L.log 2>&1; echo pt$L=$?
done
