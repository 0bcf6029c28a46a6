mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -q -m gpu -x > gpurun_out/r_tests.log 2>&1; echo tests=$?
tail -2 gpurun_out/r_tests.log
for i in 1 2; do
PSLB200_RUN_PIPELINE=0 NW=444 python tools/e2e_breakdown.py 10 2>&1 | tail -2
PSLB200_RUN_PIPELINE=1 NW=444 python tools/e2e_breakdown.py 10 2>&1 | tail -2
done
