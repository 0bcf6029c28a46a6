mkdir -p gpurun_out
A=build_ablate/lib_bandovf.so; N=paper_2107_09801_b200/libpslb200.so
python tools/ab_time.py $A $N 3 > gpurun_out/i_ab20.log 2>&1
python tools/ab_time.py $A $N 3 -- --length 262143 --walks 444 --steps 10 --mode auto > gpurun_out/i_ab18.log 2>&1
cat gpurun_out/i_ab*.log
timeout 600 python -m pytest tests/test_gpu_phase2.py tests/test_gpu_certcheck.py -q -m gpu -x > gpurun_out/i_tests.log 2>&1; echo tests=$?
