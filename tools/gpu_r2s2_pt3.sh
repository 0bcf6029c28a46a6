mkdir -p gpurun_out
for L in 16383 65535; do
  PSLB200_LIB=build_ablate/lib_pt.so timeout 300 python tools/pt_run.py 10 $L > gpurun_out/pt3_$L.log 2>&1; echo pt$L=$?
done
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --exact-steps 0 --e2e-steps 10 > gpurun_out/pt3_bench.json 2>gpurun_out/pt3_bench.err; echo bench=$?
