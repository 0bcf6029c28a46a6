mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -q -m gpu -x > gpurun_out/r_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r_tests.log
for i in 1 2; do
PSLB200_RUN_PIPELINE=0 NW=444 python tools/e2e_breakdown.py 10 2>&1 | tail -2
PSLB200_RUN_PIPELINE=1 NW=444 python tools/e2e_breakdown.py 10 2>&1 | tail -2
done
python tools/ab_time.py build_ablate/lib_nopred.so paper_2107_09801_b200/libpslb200.so 3 -- --walks 444 --steps 4 --mode exact 2>&1 | tail -2
python tools/ab_time.py build_ablate/lib_nopred.so paper_2107_09801_b200/libpslb200.so 3 -- --length 65535 --walks 444 --steps 10 --mode exact 2>&1 | tail -2
