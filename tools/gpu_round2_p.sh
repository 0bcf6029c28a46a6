mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_phase2.py tests/test_gpu_certcheck.py tests/test_gpu_cert.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/p_tests.log 2>&1; echo tests=$?
H=build_ablate/lib_head2.so; N=paper_2107_09801_b200/libpslb200.so
python tools/ab_time.py $H $N 3 > gpurun_out/p_ab20.log 2>&1
python tools/ab_time.py $H $N 3 -- --length 262143 --walks 444 --steps 10 --mode auto > gpurun_out/p_ab18.log 2>&1
python tools/ab_time.py $H $N 3 -- --length 65535 --walks 444 --steps 20 --mode auto > gpurun_out/p_ab16.log 2>&1
cat gpurun_out/p_ab*.log
