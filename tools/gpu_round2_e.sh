mkdir -p gpurun_out
PSLB200_LIB=build_ablate/lib_pt.so timeout 300 python tools/pt_run.py 10 > gpurun_out/e_pt.log 2>&1; echo pt=$?
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 --exact-steps 0 > gpurun_out/e_plain.log 2>&1; echo plain=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:run_kernel -s 3 -c 1 \
    -o gpurun_out/e_prof -f python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2 --exact-steps 0 > gpurun_out/e_ncu.log 2>&1; echo ncu=$?
