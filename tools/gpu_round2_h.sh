mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_phase2.py tests/test_gpu_certcheck.py tests/test_gpu_cert.py tests/test_gpu_parity.py -q -m gpu -x > gpurun_out/h_tests.log 2>&1; echo tests=$?
H=build_ablate/lib_head.so; W=build_ablate/lib_nowin.so; NB=build_ablate/lib_nobulk.so; NS=build_ablate/lib_nostag.so; N=paper_2107_09801_b200/libpslb200.so
python tools/ab_time.py $H $W 3 > gpurun_out/h_ab20a.log 2>&1
python tools/ab_time.py $W $NB 3 > gpurun_out/h_ab20b.log 2>&1
python tools/ab_time.py $NB $NS 3 > gpurun_out/h_ab20c.log 2>&1
python tools/ab_time.py $NS $N 3 > gpurun_out/h_ab20d.log 2>&1
python tools/ab_time.py $H $N 3 -- --length 65535 --walks 444 --steps 20 --mode auto > gpurun_out/h_ab16.log 2>&1
cat gpurun_out/h_ab*.log
