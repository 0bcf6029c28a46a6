mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_phase2.py tests/test_gpu_certcheck.py tests/test_gpu_cert.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/g_tests.log 2>&1; echo tests=$?
B=build_ablate/lib_split1.so; N=paper_2107_09801_b200/libpslb200.so
python tools/ab_time.py $B $N 3 > gpurun_out/g_ab20.log 2>&1
python tools/ab_time.py $B $N 3 -- --length 65535 --walks 444 --steps 20 --mode auto > gpurun_out/g_ab16.log 2>&1
cat gpurun_out/g_ab*.log
