mkdir -p gpurun_out
B=paper_2107_09801_b200/libpslb200_base.so; N=paper_2107_09801_b200/libpslb200.so
timeout 1200 python -m pytest tests/test_gpu_phase2.py tests/test_gpu_certcheck.py tests/test_gpu_cert.py -q -m gpu -x > gpurun_out/d_tests.log 2>&1; echo tests=$?
python tools/ab_time.py $B $N 3 > gpurun_out/d_ab20.log 2>&1
python tools/ab_time.py $B $N 3 -- --length 262143 --walks 444 --steps 10 --mode auto > gpurun_out/d_ab18.log 2>&1
python tools/ab_time.py $B $N 3 -- --length 65535 --walks 444 --steps 20 --mode auto > gpurun_out/d_ab16.log 2>&1
cat gpurun_out/d_ab*.log
