mkdir -p gpurun_out
B=build_ablate/lib_nostag2.so; N=paper_2107_09801_b200/libpslb200.so
python tools/ab_time.py $B $N 3 > gpurun_out/l_ab20.log 2>&1
python tools/ab_time.py $B $N 3 -- --length 262143 --walks 444 --steps 10 --mode auto > gpurun_out/l_ab18.log 2>&1
cat gpurun_out/l_ab*.log
PSLB200_LIB=build_ablate/lib_pt.so timeout 300 python tools/pt_run.py 10 > gpurun_out/l_pt.log 2>&1; echo pt=$?
timeout 900 python -m pytest tests/test_gpu_phase2.py tests/test_gpu_cert.py -q -m gpu -x > gpurun_out/l_tests.log 2>&1; echo tests=$?
